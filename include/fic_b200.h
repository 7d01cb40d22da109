/*
 * fic_b200.h — C ABI of the B200-native fractal-encoder hot path.
 *
 * Drop-in boundary for the reference package `fic` (arXiv 1206.4880 PIFS
 * codec).  The reference has no FFI of its own: its encoder is the Python
 * function `fic.codec.encode` (/root/reference/pkg/src/fic/codec.py:290-427),
 * whose hot loop is `_search_chunk` (codec.py:184-264).  Each entry point
 * below replaces one reference interface, cited per function.  Signatures use
 * plain pointers and sizes only; all pointers named d_* are CUDA device
 * pointers, h_* are host pointers; `stream` is a cudaStream_t (NULL = legacy
 * default stream).
 *
 * Return codes: FIC_OK, or an error code with a message available from
 * fic_last_error() (thread-local).  Argument errors reproduce the reference's
 * ValueError texts verbatim so a Python wrapper can re-raise them unchanged.
 */
#ifndef FIC_B200_H
#define FIC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FIC_ABI_VERSION 1

enum fic_status {
  FIC_OK = 0,
  FIC_EINVAL = 1, /* invalid argument (reference ValueError) */
  FIC_ECUDA = 2,  /* CUDA runtime / launch error */
  FIC_ENOMEM = 3  /* device allocation failed */
};

/* codec.py:17-18 STRATEGY_IDS */
enum fic_strategy {
  FIC_EXHAUSTIVE = 0,
  FIC_NOSEARCH = 1,
  FIC_STATIC2 = 2,
  FIC_DYNAMIC_FD = 3
};

enum fic_fd_source { FIC_FD_ORIGINAL = 0, FIC_FD_DOWNSAMPLED = 1 };

enum fic_matcher {
  FIC_MATCH_AUTO = 0,    /* tcgen05 tensor-core screen + exact fp64 rescoring;
                            small pools on the exact path */
  FIC_MATCH_EXACT = 1    /* exact fp64 evaluation of every candidate (CUDA cores) */
};

/* Packed transform record, codec.py:24-26 RECORD_DTYPE (7 bytes, LE). */
#pragma pack(push, 1)
typedef struct fic_record {
  uint32_t domain;   /* raster domain index */
  uint8_t isometry;  /* 0..7, blocks.py:113-124 */
  uint8_t s_q;       /* 0..31 */
  uint8_t o_q;       /* 0..127 */
} fic_record_t;
#pragma pack(pop)

/* Arguments of codec.encode (codec.py:290-300) plus the fixed-window
 * extension `delta` and range sharding. */
typedef struct fic_params {
  int32_t range_size;   /* default 8 */
  int32_t domain_size;  /* must be 2*range_size */
  int32_t stride;       /* >= 1 */
  int32_t isometries;   /* 0: identity only, 1: all 8 */
  int32_t strategy;     /* enum fic_strategy */
  int32_t fd_source;    /* enum fic_fd_source */
  int32_t has_delta;    /* 1: window half-width = delta; 0: D_f = (max-min)/3 */
  int32_t matcher;      /* enum fic_matcher */
  double delta;
  /* ln(k) for k = 0..ln_len-1 as computed by the caller's numpy (fdim.py:76
   * uses np.log; passing the caller's table keeps FD bit-identical to the
   * caller's own reference).  NULL: the library uses C log(). */
  const double* h_ln_table;
  int32_t ln_len;
  /* Range sharding: this call matches only ranges whose position in the
   * cost-balanced FD-sorted order falls in shard `shard_index` of
   * `shard_count`.  Other ranges' outputs are left untouched.  1-of-1 = all. */
  int32_t shard_index;
  int32_t shard_count;
  int32_t max_segment;  /* columns per work item (0 = library default) */
  int32_t small_pool;   /* ranges with fewer candidates use the exact path (0 = default) */
  /* DBC slope weights (fdim.py:37-41) for the domain-FD block side and the
   * range side, as the caller's numpy computes them; NULL = computed in C. */
  const double* h_fd_weights_dom;
  const double* h_fd_weights_rng;
  int32_t n_fd_weights_dom, n_fd_weights_rng;
} fic_params_t;

/* EncodeStats fields (codec.py:77-87) plus device-side diagnostics. */
typedef struct fic_stats {
  int64_t n_ranges;
  int64_t n_domains;
  int64_t comparisons;       /* sum(pool) * n_iso over ALL ranges (codec.py:419) */
  double mean_pool_size;     /* codec.py:420 */
  double fd_min, fd_max;     /* fd_stats over domain FDs (fdim.py:93-100) */
  double half_width;         /* D_f or delta (dynamic_fd), else 0 */
  double ms_fd;              /* device time of FD + index + window build */
  double ms_pool;            /* device time of pool builder */
  double ms_match;           /* device time of the matcher kernels (tensor + exact + merge) */
  double ms_tensor;          /* device time of the tcgen05 matcher launch */
  double ms_exact;           /* device time of the exact-path matcher launch */
  double ms_total;           /* device time of the whole call */
  int64_t exact_evals;       /* candidates evaluated in fp64 (survivors + exact path) */
  int64_t tensor_candidates; /* candidates screened on the tensor cores (incl. masked padding) */
  int64_t tensor_comparisons; /* useful candidates of tensor-path ranges: sum(pool) * n_iso */
  int32_t tensor_tiles, exact_tiles, work_items;
  int32_t kernel_launches;   /* kernels this call launched (library-internal CUB passes excluded) */
  double ms_pool_main;       /* device time of the pool builder's main kernel (k_pool) alone */
  int64_t graph;             /* 0 enqueued directly, 1 recorded as a CUDA graph and launched, 2 replayed */
  double ms_sl;              /* device time of the survivor-list and hit-list rescoring (k_sl_rescore, k_hl_rescore) */
  int64_t sl_entries;        /* survivor-list entries (row, 64-column chunk, mask) rescored after the matcher */
  int64_t hl_entries;        /* hit-list entries (warp of rows, 64-column chunk, hit ballot) rescored after the matcher */
  int64_t hl_tests;          /* hit-list candidates tested against the exact lower bound */
} fic_stats_t;

/* Replaces fic.codec.encode (codec.py:290-427) for one image already in
 * device memory.  Outputs (caller-allocated, device, R = (h/rs)*(w/rs)):
 * d_records R*7 bytes, d_pre_rms/d_post_rms R doubles, d_pool_sizes R int64
 * (may be NULL).  h_stats may be NULL.  Synchronises `stream` once at the end
 * (stats read-back). */
int fic_encode_v1(const uint8_t* d_image, int32_t height, int32_t width,
                  const fic_params_t* params, uint8_t* d_records,
                  double* d_pre_rms, double* d_post_rms, int64_t* d_pool_sizes,
                  fic_stats_t* h_stats, void* stream);

/* Pool plan only (FD, FD index, per-range slabs) — the setup half of encode
 * (codec.py:343-375; fdim.dbc_grid fdim.py:44-80; AvlTree.as_sorted_arrays
 * avltree.py:150-189).  Device outputs, any may be NULL:
 * d_fd_dom[D], d_fd_rng[R] (dynamic_fd/static2 only), d_order[D] (raster id
 * of each pool-ordered domain), d_slab_lo[R], d_slab_hi[R]. */
int fic_plan_v1(const uint8_t* d_image, int32_t height, int32_t width,
                const fic_params_t* params, double* d_fd_dom, double* d_fd_rng,
                int64_t* d_order, int64_t* d_slab_lo, int64_t* d_slab_hi,
                fic_stats_t* h_stats, void* stream);

/* The pool builder alone (K1) -- fic.blocks.downsample2(domain_stack)
 * (blocks.py:75-82, 158-164) and the _SearchContext sums (codec.py:136-157),
 * in the pool order of `params` (FD order for dynamic_fd / static2, raster
 * otherwise; codec.py:159-164 use_order).  Device outputs, any may be NULL:
 * d_order[D] raster domain id per pool position, d_decimated[D*K] uint8,
 * d_sums[2*D] uint32 (sum_d, sum_dd) pairs, d_inv_den[D] (1/den, 0 where
 * den == 0), d_b_rows[D*K] fp16 bits of the tensor path's centred unit-norm
 * rows (K = 16 or 64 only).  Synchronises `stream`. */
int fic_pool_v1(const uint8_t* d_image, int32_t height, int32_t width,
                const fic_params_t* params, int64_t* d_order, uint8_t* d_decimated,
                uint32_t* d_sums, double* d_inv_den, uint16_t* d_b_rows, void* stream);

/* Replaces fic.fdim.dbc_grid (fdim.py:44-80) for an (n, side, side) uint8
 * stack in device memory; d_fd[n] receives the dimension (clamped to [2,3]
 * when clamp != 0). */
int fic_dbc_v1(const uint8_t* d_blocks, int64_t n, int32_t side, int32_t clamp,
               const double* h_ln_table, int32_t ln_len, const double* h_weights,
               int32_t n_weights, double* d_fd, void* stream);
/* The same with the reference's gray_levels argument (fdim.py:45, 74: box
 * height h = s * gray_levels / side); fic_dbc_v1 is gray_levels = 256. */
int fic_dbc_v2(const uint8_t* d_blocks, int64_t n, int32_t side, int32_t gray_levels,
               int32_t clamp,
               const double* h_ln_table, int32_t ln_len, const double* h_weights,
               int32_t n_weights, double* d_fd, void* stream);

/* Replaces fic.codec.decode (codec.py:516-598): `iterations` passes from a
 * constant gray level `initial` (128 in the reference), or from d_initial
 * (h*w uint8, may be NULL).  d_out receives the final uint8 image. */
int fic_decode_v1(const uint8_t* d_records, int32_t height, int32_t width,
                  int32_t range_size, int32_t domain_size, int32_t stride,
                  int32_t iterations, double initial, const uint8_t* d_initial,
                  uint8_t* d_out, void* stream);

/* One pass of fic.codec.decode_iterates (codec.py:534-598): d_dst[h*w] =
 * the next float64 iterate computed from d_src[h*w]; d_out (optional, h*w
 * uint8) receives rint(d_dst), the snapshot decode_iterates yields.
 * Isometry bytes > 7 keep the identity as in the reference; records are not
 * re-validated here (fic_decode_v1 / the Python layer do that first), an
 * out-of-geometry domain index reads domain 0 instead of faulting. */
int fic_decode_step_v1(const uint8_t* d_records, int32_t height, int32_t width,
                       int32_t range_size, int32_t domain_size, int32_t stride,
                       const double* d_src, double* d_dst, uint8_t* d_out, void* stream);

/* Multi-GPU range sharding exchange (replaces the reference's per-thread
 * result slots, codec.py:386-397, across processes).  pack: the rank's
 * outputs (ranges it matched have post RMS >= 0) as an int64 [n][3] buffer
 * -- record bytes | owner count << 56, pre RMS bits, post RMS bits -- zero
 * elsewhere, for one all-reduce (SUM) over the ranks.  unpack: the reduced
 * buffer back into records / RMS; *d_bad = ranges whose owner count != 1. */
int fic_shard_pack_v1(const uint8_t* d_records, const double* d_pre_rms, const double* d_post_rms,
                      int64_t n, int64_t* d_buf, void* stream);
int fic_shard_unpack_v1(const int64_t* d_buf, int64_t n, uint8_t* d_records, double* d_pre_rms,
                        double* d_post_rms, uint32_t* d_bad, void* stream);

/* Diagnostic: with FIC_ARENA_GUARD set in the environment every scratch buffer
 * of a call is followed by a red zone that is verified after the call's
 * kernels (a write check for boxes without compute-sanitizer; the call fails
 * with FIC_ECUDA and a message naming the buffer).  This entry exercises the
 * check itself on the current device: a 1000-byte scratch buffer is filled
 * with `overrun` extra bytes.  Returns FIC_OK when the zones are intact (or
 * the guard is off), FIC_ECUDA when the overrun was caught.  No reference
 * counterpart (the reference is pure numpy). */
int fic_guard_selftest_v1(int32_t overrun);

const char* fic_last_error(void);
int fic_abi_version(void);
/* Releases cached device workspaces of the calling thread's current device. */
void fic_release(void);

#ifdef __cplusplus
}
#endif
#endif /* FIC_B200_H */
