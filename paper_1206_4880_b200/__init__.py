"""B200-native fractal-image encoder hot path (arXiv 1206.4880), see DESIGN.md.

Public names mirror the reference package ``fic`` for the rebuilt path:
``encode``, ``decode``, ``decode_iterates``, ``serialize``, ``deserialize``,
``FractalCode``, ``EncodeStats``, ``FormatError``, ``RECORD_DTYPE``,
``dbc_grid``, ``dbc_dimension``, ``dbc_dimension_raw``, ``fd_stats``, ``FdStats``,
``scale_set``, ``fit_transform``, ``quantize_so``, ``dequantize_so``.
"""

from .codec import (  # noqa: F401
    RECORD_DTYPE,
    STRATEGIES,
    STRATEGY_IDS,
    EncodeStats,
    FdStats,
    FormatError,
    FractalCode,
    dbc_dimension,
    dbc_dimension_raw,
    dbc_grid,
    decode,
    decode_iterates,
    dequantize_so,
    deserialize,
    encode,
    encode_device,
    fd_stats,
    fit_transform,
    plan,
    quantize_so,
    scale_set,
    serialize,
)

__version__ = "0.1.0"
