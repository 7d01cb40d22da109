// Matcher launchers (internal interface).
#pragma once
#include "common.cuh"

namespace fic {

// Where the matchers read a domain's decimated pixels (blocks.py:75-82).
// The pool builder does not write a per-pool-position copy of them: the
// rescorers and the exact matcher gather a domain by raster id from the
// pool builder's own L2-resident intermediates.
struct DomSrc {
  const unsigned long long* trows;  // RS 8: [ndx][2][mh] row segments; domain (Y, X) =
                                    // 8 consecutive words at (dx * 2 + (Y & 1)) * mh + (Y >> 1)
  const uint8_t* planes;            // RS 4/8: [2][plane_rows][pitch] box-floor planes
  const uint8_t* raw;               // other sizes: [D][KP] pool order, rows zero-padded to KP
  int ndx, st, mh, plane_rows, pitch;
  int KP;                           // raw row pitch (K rounded up to a multiple of 4)
};

// Column (domain) data in pool order, produced by the pool builder (K1).
struct PoolView {
  const uint16_t* bh;      // [D][K] fp16 bits (tensor path)
  const double* inv_den;   // [D]
  const uint2* sums;       // [D] (sum_d, sum_dd)
  const uint32_t* order;   // [D] raster domain index per pool position (nullptr = identity)
  DomSrc src;
  int64_t D;
};

__device__ __forceinline__ uint32_t pool_id(const PoolView& P, int64_t p) {
  return P.order ? __ldg(P.order + p) : (uint32_t)p;
}

// 4 bytes starting at byte address q (4-byte aligned loads + funnel shift)
__device__ __forceinline__ uint32_t bytes4_at(const uint8_t* q) {
  const uintptr_t u = reinterpret_cast<uintptr_t>(q);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(u & ~(uintptr_t)3);
  return __funnelshift_r(__ldg(w), __ldg(w + 1), (uint32_t)(u & 3) * 8);
}

// The K/4 little-endian words of the decimated domain at pool position p
// (raster id `id`), K = 64 or 16 (RS 8 / 4).  SRC selects the source at
// compile time (the tensor matcher is instantiated per source: a runtime
// three-way branch in its inlined rescoring costs the screeners registers);
// SRC_ANY branches at run time (exact matchers, tests).
enum { SRC_TROWS = 0, SRC_PLANES = 1, SRC_RAW = 2, SRC_ANY = 3 };

template <int K, int SRC = SRC_ANY>
__device__ __forceinline__ void dom_words(const PoolView& P, int64_t p, uint32_t id,
                                          uint32_t (&w)[K / 4]) {
  constexpr int RS = K == 64 ? 8 : 4;
  const DomSrc& d = P.src;
  const uint32_t dy = id / (uint32_t)d.ndx, dx = id - dy * (uint32_t)d.ndx;
  const uint32_t Y = dy * d.st, X = dx * d.st;
  if (RS == 8 && (SRC == SRC_TROWS || (SRC == SRC_ANY && d.trows))) {
    const unsigned long long* t = d.trows + ((size_t)dx * 2 + (Y & 1)) * d.mh + (Y >> 1);
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const unsigned long long v = __ldg(t + i);
      w[2 * i] = (uint32_t)v;
      w[2 * i + 1] = (uint32_t)(v >> 32);
    }
  } else if (SRC == SRC_PLANES || (SRC == SRC_ANY && d.planes)) {
    const uint8_t* b = d.planes + (size_t)(X & 1) * d.plane_rows * d.pitch + (size_t)Y * d.pitch +
                       (X >> 1);
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      if (RS == 8) {
        const uint8_t* q = b + (size_t)(2 * i) * d.pitch;
        w[2 * i] = bytes4_at(q);
        w[2 * i + 1] = bytes4_at(q + 4);
      } else {
        w[i] = bytes4_at(b + (size_t)(2 * i) * d.pitch);
      }
    }
  } else {
    const uint4* q = reinterpret_cast<const uint4*>(d.raw + (size_t)p * K);
#pragma unroll
    for (int i = 0; i < K / 16; ++i) {
      const uint4 v = __ldg(q + i);
      w[4 * i] = v.x;
      w[4 * i + 1] = v.y;
      w[4 * i + 2] = v.z;
      w[4 * i + 3] = v.w;
    }
  }
}

// Range data (raster index).
struct RangeView {
  const RangeInfo* info;   // [R]
  const uint8_t* rows;     // [R][n_iso][KP] permuted pixels (rows zero-padded to KP)
  const int32_t* lo;       // [R] slab start (pool order)
  const int32_t* hi;       // [R] slab end
  int n_iso, K, KP;        // KP: row pitch, K rounded up to a multiple of 4
};

// Work counts of one encode, computed on the device by the planner
// (k_plan_scans) and read by the matchers: the host enqueues everything
// without waiting for them (its allocations use upper bounds).
struct DevPlan {
  int64_t tb, n_tr, n_tt;      // tensor ranges: first sorted position, count, tiles
  int64_t eb, n_er;            // exact ranges: first sorted position, count
  int64_t n_titems, n_eitems, n_slots;
  int64_t n_split;             // tensor items run as pieces (tail splitting)
};

// Exact CUDA-core matcher: one work item = (range, segment of its slab).
struct ExactArgs {
  const int2* items;           // (index into elist, segment)
  int64_t n_items;
  const uint32_t* elist;       // range ids of the exact class (this shard)
  int seg_len;
  const int64_t* slot_base;    // [R]
  Partial* partials;
  unsigned long long* counters;  // [0] exact evaluations
  const DevPlan* plan;         // non-null: n_items = plan->n_eitems, elist += plan->eb (n_items: bound)
};
void launch_exact(const PoolView& P, const RangeView& Rv, const ExactArgs& a,
                  cudaStream_t s);

// Tensor-core matcher: one work item = (tile of RT ranges x n_iso rows,
// segment of the tile's union window).
struct TcArgs {
  const int2* items;           // (tile, segment)
  int64_t n_items;
  const uint32_t* tlist;       // range ids of the tensor class (this shard), tile order
  int64_t n_tr;
  const int32_t* wlo;          // [tiles] union window
  const int32_t* whi;
  int seg_len;                 // columns per work item (segments >= 1)
  int seg0;                    // columns of a tile's first segment (short: it seeds the thresholds)
  int RT;                      // ranges per tile = 128 / n_iso
  const int64_t* slot_base;
  Partial* partials;
  unsigned long long* counters;  // [0] exact evaluations, [1] screened candidates
  unsigned long long* item_ctr;  // dynamic work-item counter (zeroed before the launch)
  unsigned long long* thr_g;   // [R] best exact error so far per range (double bits), shared by
                               // the items (segments) of a range; any value is a valid bound
  int debug;                   // FIC_TC_DEBUG (timing experiments only; results invalid if != 0)
  unsigned long long* dbg;     // timeline buffer (debug & 32)
  int64_t n_split;             // the last n_split items run as nsub column pieces each
  int nsub;                    // partial slots per segment (slot = segment * nsub + piece)
  // flat ranges (all pixels equal) whose slab is the canonical flat slab are
  // matched by the flat kernels (fic_flat.cu), not screened: nullptr = none
  const int16_t* flat_c;       // [R] pixel value of a flat range, -1 otherwise
  const uint32_t* flat_canon;  // [1] smallest flat range index (its slab is canonical)
  const DevPlan* plan;         // non-null: n_items / n_tr / n_split / tlist offset from the device
  // Survivor list: a hit chunk whose row queue cannot take its survivors
  // writes one 16-byte entry (range id << 3 | isometry, pool column of bit
  // 0, 64-bit survivor mask) here instead of waiting for the rescoring warp;
  // k_sl_rescore evaluates them after the matcher.  nullptr = off.
  uint4* sl;
  uint32_t* sl_count;          // [1] entries handed out in per-warp chunks (unused chunk tails hold
                               // empty entries; may exceed sl_cap: the rest were queued)
  uint32_t sl_cap;
  int pilot_cols;              // > 0: one pilot item per tile first (the first pilot_cols columns of its
                               // window): per row the PK largest |u|, evaluated exactly, seed the
                               // ranges' thresholds (thr_g) for the main items
  int pilot_stride;            // pilot items sample every pilot_stride-th 128-column tile (>= 1);
                               // 0: adaptive, about pilot_samples tiles of each window
  int pilot_samples;
  int sl_all;                  // 1: every survivor goes to the list (the queues carry seeds only);
                               // 2: the same after each tile's first segment (a pilot with the queues)
  // Hit list (with sl_all == 1): a screening warp whose chunk has any lane
  // with max |u| over the row's threshold writes ONE 16-byte entry (tlist
  // index of the tile's first range, first row of the warp, pool column of
  // the chunk, 32-bit ballot of the hit rows) instead of building per-row
  // survivor masks; k_hl_rescore filters those chunks with the exact
  // integer lower bound and evaluates the rest.  nullptr = off.
  uint4* hl;
  uint32_t* hl_count;          // [1] entries handed out in per-warp chunks (tails: empty entries)
  uint32_t hl_cap;
};

// Rescoring of the survivor list: every candidate of every entry, exactly;
// per-range lexicographic (err, dom, iso) minimum by a 128-bit CAS on
// best[r] = {dom << 32 | iso << 24 | s_q << 16 | o_q << 8, err bits} and the
// pre-quantisation minimum by a 64-bit atomicMin on pre[r].
struct SlArgs {
  const uint4* sl;
  const uint32_t* sl_count;
  uint32_t sl_cap;
  unsigned long long* best;    // [R][2]
  unsigned long long* pre;     // [R]
  unsigned long long* counters;  // [0] exact evaluations
};
void launch_sl_rescore(const PoolView& P, const RangeView& Rv, const SlArgs& a, cudaStream_t s);

// Rescoring of the hit list (TcArgs::hl): one warp per entry, two chunk
// columns per lane; for every hit row, each column of the row's slab whose
// exact lower bound V - num^2 / (K den) (num = K cross - sum_r sum_d, den =
// K sum_dd - sum_d^2, integers) can reach the range's threshold is evaluated
// with eval_candidate into the survivor list's best / pre arrays.
struct HlArgs {
  const uint4* hl;
  const uint32_t* hl_count;
  uint32_t hl_cap;
  const uint32_t* tlist;       // the tensor matcher's tlist (plan offset applied here)
  const DevPlan* plan;
  const unsigned long long* thr_g;  // [R] thresholds from the matcher (double bits)
  unsigned long long* best;    // [R][2] (SlArgs::best)
  unsigned long long* pre;     // [R]
  unsigned long long* counters;  // [0] exact evaluations
  unsigned long long* tests;     // [1] lower-bound tests
  // sorted copy (launch_hl_sort; nullptr: read the list as written)
  const uint4* sorted;         // [hl_cap] entries ordered by chunk column / 64
  const uint32_t* n_sorted;    // [1] entries in `sorted`
  uint32_t* bins;              // [D / 64 + 2] histogram -> cursors
  uint32_t* run_ctr;           // [1] runs of the sorted list handed out (zeroed per call)
};
void launch_hl_sort(const HlArgs& a, int64_t D, cudaStream_t s);
void launch_hl_rescore(const PoolView& P, const RangeView& Rv, const HlArgs& a, cudaStream_t s);



// Flat ranges (every pixel equal to c): all isometries give the same row and
// the LS fit is s = 0, o = c exactly, so each candidate's error is a function
// of (c, sum_d, sum_dd) alone and the range's best is shared by all flat
// ranges with the same value and slab -- one reduction per value c instead
// of a screen that cannot prune them (its lower bound V - u^2 is 0).
struct FlatArgs {
  const uint8_t* img;
  int W, rs, nrx, R;
  int16_t* flat_c;             // [R] out (detect): c or -1
  unsigned long long* n_flat;  // [1] out (detect): count
  uint32_t* canon;             // [1] out (detect): smallest flat range index (init 0xffffffff)
  const int32_t* lo;           // [R] slabs
  const int32_t* hi;
  const int32_t* nslots;       // [R] ranges matched by this call (> 0)
  uint8_t* present;            // [256] values of canonical flat ranges matched here
  struct Best { double err; uint32_t dom; int32_t sq, oq, pad; };
  Best* part;                  // [256][nchunk] per-chunk bests
  Best* best;                  // [256]
  int nchunk;
  int64_t D;
  int K;
  uint8_t* records;
  double* pre_rms;
  double* post_rms;
};
void launch_flat_detect(const FlatArgs& a, cudaStream_t s);
void launch_flat_match(const PoolView& P, const FlatArgs& a, cudaStream_t s);
bool tc_supported(int K);
int tc_tile_rows(int K);
void launch_tc(const PoolView& P, const RangeView& Rv, const TcArgs& a, cudaStream_t s);

// Merge partial bests into records + RMS (codec.py:259-264, 399-405).
struct MergeArgs {
  int R;
  const int64_t* slot_base;    // [R]
  const int32_t* nslots;       // [R] (0 = not matched in this call)
  const Partial* partials;
  uint8_t* records;            // [R][7]
  double* pre_rms;
  double* post_rms;
  double n;                    // pixels per range
  const unsigned long long* sl_best;  // optional [R][2] (SlArgs)
  const unsigned long long* sl_pre;   // [R]
  unsigned long long* err_out;  // optional [R]: each range's best error bits (FIC_PRIME_THR experiment)
};
void launch_merge(const MergeArgs& a, cudaStream_t s);

}  // namespace fic
