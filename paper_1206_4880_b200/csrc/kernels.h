// Host-side launchers of the library's kernels (internal interface).
#pragma once
#include "common.cuh"

namespace fic {

// ---- K2: differential box counting (fdim.py:44-80) -------------------------
enum FdMode { FD_IMAGE = 0, FD_DECIMATED = 1, FD_STACK = 2 };
struct FdArgs {
  const uint8_t* src;   // image (modes 0/1) or block stack (mode 2)
  int W;                // image width (modes 0/1)
  int side;             // block side M
  int bst;              // block origin step in image pixels (modes 0/1)
  int nbx;              // blocks per row (modes 0/1)
  int64_t n;            // blocks
  int mode;
  int clamp;
  int J;                // number of DBC scales (2..7)
  int smax;             // coarsest scale
  const uint16_t* quot; // [J][256] floor(v / h_j) (host-built, fdim.py:74-75)
  const double* ln;     // ln table (fdim.py:76 np.log)
  int ln_len;
  const double* w;      // [J] slope weights
  double* fd;           // [n] output
  unsigned long long* key;  // [n] optional: fd bits for sorting
  uint32_t* combo;          // [n] optional: index of the count combination (k_fd<SMAX> only)
  int cstride[7];           // combination index stride per scale (0 = scale not indexed)
  const uint32_t* rank_of_combo;  // optional [C]: write rank_of_combo[combo] to `rank`
  uint32_t* rank;                 // [n] (with rank_of_combo; replaces combo)
  uint32_t* iota;                 // [n] optional: iota[b] = b (sort payload)
  int qshift[7];                  // floor(v / h_j) == v >> qshift[j] for all v (else -1)
  uint32_t* rank_hist;            // optional [n_rank]: global histogram of `rank` (atomics)
  uint32_t* rank_minid;           // with rank_hist [n_rank]: smallest block index per rank
  int n_rank;
};
// Builds host-side tables for block side `side` into `quot` (J*256), returns
// J and the coarsest scale and the ln-table length required.
int dbc_tables(int side, uint16_t* quot, int* smax, int* ln_needed, int gray_levels = 256);
void launch_fd(const FdArgs& a, cudaStream_t s);

// ---- K3: FD index + slabs (avltree.py:150-189, codec.py:343-375) ------------
struct SlabArgs {
  const double* keys;      // sorted domain FDs (pool order); nullptr = rank form below
  // rank form (compact FD sort): rank_start[r] = first pool position with
  // rank >= r (r <= n_rank), key of pool position p = fd_of_rank[rank of p]
  const double* fd_of_rank;
  const uint32_t* rank_start;
  int n_rank;
  const uint32_t* ids;     // raster id per pool position
  const double* fd_rng;    // [R]
  int64_t D;
  int R;
  int strategy;
  int has_delta;
  double delta;
  double* scal;            // [4] out: f_min, f_max, half / mid, boundary
  int scal_ready;          // scal already written (by the counting sort's scan)
  uint32_t* lo_rank;       // [R] optional (rank form, dynamic_fd): rank index q with lo = rank_start[q]
  int32_t* lo;             // [R] out
  int32_t* hi;             // [R] out
  // geometry for nosearch (codec.py:430-447)
  int H, W, rs, ds, st, nrx, ndx;
};
void launch_slabs(const SlabArgs& a, cudaStream_t s);
void launch_rank_start(const uint32_t* rks, int64_t D, int n_rank, uint32_t* start,
                       cudaStream_t s);
// Counting sort by rank (ranks < n_rank <= kCountSortMaxRanks): hist and
// minid (from launch_fd) -> start/cursor, scatter.  Each bucket starts with
// its smallest index, the rest of a bucket is in unspecified order.
constexpr int kCountSortMaxRanks = 8192;
struct ScalArgs {          // slab scalars computed by the counting sort's scan (optional)
  const double* fd_of_rank;
  int strategy, has_delta;
  double delta;
  double* scal;            // nullptr = skip
};
void launch_count_sort(const uint32_t* rank, int64_t D, int n_rank, const uint32_t* hist,
                       const uint32_t* minid, uint32_t* start, uint32_t* cursor, uint32_t* order,
                       const ScalArgs& sa, cudaStream_t s);

// ---- K1: pool builder (blocks.py:75-82, codec.py:136-145) -------------------
struct PoolArgs {
  const uint8_t* img;
  int H, W, rs, st, ndx;
  uint8_t* planes;         // [2][plane_rows][pitch] box-floor planes (scratch)
  int plane_rows, pitch;
  unsigned long long* trows;  // optional (RS = 8): [ndx][2][mh] decimated row segments, so a
  int mh;                     // domain's 8 rows are 64 contiguous bytes (scratch)
  int64_t D;
  const uint32_t* order;   // raster id per pool position (nullptr = identity)
  uint8_t* raw;            // generic sizes only: [D][KP] decimated pixels, pool order, zero-padded
  int KP;                  // raw row pitch
  uint16_t* bh;            // [D][K] fp16 centred unit-norm rows (nullptr = skip)
  double* inv_den;         // [D]
  uint2* sums;             // [D] (sum_d, sum_dd)
  cudaEvent_t ev_main;     // optional: recorded just before the main kernel (k_pool)
};
void launch_pool(const PoolArgs& a, cudaStream_t s);

// ---- range preparation -------------------------------------------------------
struct RangeArgs {
  const uint8_t* img;
  int W, rs, nrx, R, n_iso;
  const int* inv_perm;     // [8][K] device
  RangeInfo* info;         // [R]
  uint8_t* rows;           // [R][n_iso][KP] permuted range pixels (zero-padded rows)
  int KP;
};
void launch_ranges(const RangeArgs& a, cudaStream_t s);

// ---- planning -----------------------------------------------------------------
struct PlanCounts {        // read back to the host once
  int64_t shard_begin, shard_end;  // sorted positions of this shard
  int64_t n_tensor;                // ranges of the tensor class (all shards)
  int64_t pool_sum;                // sum(pool) over all ranges
};

}  // namespace fic
