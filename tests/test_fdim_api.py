"""The fdim API surface (fdim.py:19-100) against vectors the reference itself
produced (tests/golden/make_fdim_golden.py): gray_levels other than 256,
dbc_dimension / dbc_dimension_raw, fd_stats, scale_set."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import fic_oracle as orc
from paper_1206_4880_b200 import codec

G = load_golden("fdim_api_cases.npz")
SIDES = (8, 12, 16, 24)
GRAYS = (64, 128, 256, 512, 1000)


@pytest.mark.parametrize("side", SIDES)
def test_oracle_dbc_gray_levels_match_reference(side):
    blocks = G[f"s{side}.blocks"]
    for gray in GRAYS:
        assert np.array_equal(orc.dbc(blocks, gray), G[f"s{side}.g{gray}.fd"])
        assert np.array_equal(orc.dbc(blocks, gray, clamp=False), G[f"s{side}.g{gray}.raw"])


def test_host_mirrors_match_reference():
    st = codec.fd_stats(G["stats.fds"])
    assert [st.f_min, st.f_max, st.d_f] == list(G["stats.out"])
    assert isinstance(st, codec.FdStats)
    with pytest.raises(ValueError, match="fd_stats requires a non-empty sequence"):
        codec.fd_stats([])
    assert [len(codec.scale_set(s)) for s in range(1, 65)] == list(G["scale_sets"])
    assert codec.scale_set(16) == [2, 4, 8] and codec.scale_set(12) == [2, 4]


@pytest.mark.gpu
@pytest.mark.parametrize("side", SIDES)
def test_gpu_dbc_gray_levels_match_reference(side):
    blocks = G[f"s{side}.blocks"]
    for gray in GRAYS:
        assert np.array_equal(codec.dbc_grid(blocks, gray), G[f"s{side}.g{gray}.fd"]), gray
        assert np.array_equal(codec.dbc_grid(blocks, gray, clamp=False), G[f"s{side}.g{gray}.raw"]), gray
        assert np.array_equal(codec.dbc_grid(blocks, gray_levels=gray, clamp=True), G[f"s{side}.g{gray}.fd"])
    assert [codec.dbc_dimension(b) for b in blocks[:8]] == list(G[f"s{side}.dim"])
    assert [codec.dbc_dimension_raw(b, 128) for b in blocks[:8]] == list(G[f"s{side}.dim_raw"])


@pytest.mark.gpu
def test_gpu_dbc_rejects_what_it_cannot_take():
    with pytest.raises(ValueError, match="expected an \\(n, M, M\\) stack of square blocks"):
        codec.dbc_grid(np.zeros((2, 8, 4), np.uint8))
    with pytest.raises(ValueError, match="block side 4 too small: need at least two DBC scales"):
        codec.dbc_grid(np.zeros((1, 4, 4), np.uint8))
    with pytest.raises(ValueError, match="uint8"):
        codec.dbc_grid(np.zeros((1, 8, 8), np.uint16))
    with pytest.raises(ValueError, match="gray_levels"):
        codec.dbc_grid(np.zeros((1, 8, 8), np.uint8), 0)
