// Exact CUDA-core matcher (K5 on whole slabs) and the partial merge (K6).
//
// Every candidate (range, domain, isometry) of a work item is evaluated with
// the reference's fp64 op sequence (codec.py:218-242, see eval_candidate):
// the cross term is an exact integer dot product (u8 x u8 via dp4a), every
// fp64 op is an explicit round-to-nearest intrinsic (no FMA), so results are
// bit-identical to numpy's.  Used for small pools (fallback ranges, nosearch)
// and as the device-side oracle (FIC_MATCH_EXACT).
#include <algorithm>

#include "match.h"

namespace fic {

struct Best {
  double err, pre;
  uint32_t dom;
  int iso, sq, oq;
};

__device__ __forceinline__ void best_init(Best& b) {
  b.err = INFINITY;
  b.pre = INFINITY;
  b.dom = 0xffffffffu;
  b.iso = 0;
  b.sq = 0;
  b.oq = 0;
}

__device__ __forceinline__ void best_merge(Best& a, const Best& b) {
  if (better(b.err, b.dom, b.iso, a.err, a.dom, a.iso)) {
    a.err = b.err;
    a.dom = b.dom;
    a.iso = b.iso;
    a.sq = b.sq;
    a.oq = b.oq;
  }
  a.pre = fmin(a.pre, b.pre);
}

__device__ __forceinline__ Best shfl_best(const Best& b, int lane_mask) {
  Best o;
  o.err = __shfl_xor_sync(0xffffffffu, b.err, lane_mask);
  o.pre = __shfl_xor_sync(0xffffffffu, b.pre, lane_mask);
  o.dom = __shfl_xor_sync(0xffffffffu, b.dom, lane_mask);
  o.iso = __shfl_xor_sync(0xffffffffu, b.iso, lane_mask);
  o.sq = __shfl_xor_sync(0xffffffffu, b.sq, lane_mask);
  o.oq = __shfl_xor_sync(0xffffffffu, b.oq, lane_mask);
  return o;
}

// Every candidate of range r against pool columns [c0, c1), one thread per
// column (all isometries), block-wide lexicographic best.  The block has
// staged the range's n_iso permuted rows in srow.  Returns the block's best
// in thread 0 and adds the evaluations to counters[0].
template <int K>
__device__ __forceinline__ Best scan_columns(const PoolView& P, const RangeView& Rv, uint32_t r,
                                             int64_t c0, int64_t c1,
                                             const uint32_t (*srow)[K / 4], Best* sbest,
                                             unsigned long long* counters) {
  constexpr int KW = K / 4;
  const RangeInfo inf = Rv.info[r];
  const double n = (double)K;
  const int n_iso = Rv.n_iso;
  Best b;
  best_init(b);
  unsigned long long evals = 0;
  for (int64_t p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
    const uint32_t dom = pool_id(P, p);
    uint32_t dw[KW];
    dom_words<K>(P, p, dom, dw);
    uint2 sm = P.sums[p];
    double sd = (double)sm.x, sdd = (double)sm.y, inv = P.inv_den[p];
    for (int i = 0; i < n_iso; ++i) {
      uint32_t acc = 0;
#pragma unroll
      for (int q = 0; q < KW; ++q) acc = __dp4a(dw[q], srow[i][q], acc);
      Cand c = eval_candidate((double)acc, sd, sdd, inv, inf.sr, inf.srr, n);
      b.pre = fmin(b.pre, c.pre);
      if (better(c.err, dom, i, b.err, b.dom, b.iso)) {
        b.err = c.err;
        b.dom = dom;
        b.iso = i;
        b.sq = c.sq;
        b.oq = c.oq;
      }
    }
    evals += n_iso;
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) best_merge(b, shfl_best(b, m));
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sbest[warp] = b;
  for (int m = 16; m >= 1; m >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, m);
  if (lane == 0 && evals) atomicAdd(counters, evals);
  __syncthreads();
  Best t = sbest[0];
  if (threadIdx.x == 0)
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best_merge(t, sbest[w]);
  return t;
}

__device__ __forceinline__ Partial to_partial(const Best& t, bool valid) {
  Partial out;
  out.err = t.err;
  out.pre = t.pre;
  out.dom = t.dom;
  out.iso = (uint8_t)t.iso;
  out.sq = (uint8_t)t.sq;
  out.oq = (uint8_t)t.oq;
  out.valid = valid ? 1 : 0;
  return out;
}

template <int K>
__global__ void __launch_bounds__(256) k_exact(PoolView P, RangeView Rv, ExactArgs a) {
  constexpr int KW = K / 4;  // 32-bit words per row
  __shared__ uint32_t srow[8][KW];
  __shared__ Best sbest[8];
  int64_t n_items = a.n_items;
  const uint32_t* elist = a.elist;
  if (a.plan) {  // device-side work count (n_items is then a bound)
    n_items = a.plan->n_eitems;
    elist = a.elist + a.plan->eb;
  }
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    int2 item = a.items[it];
    uint32_t r = elist[item.x];
    int64_t lo = Rv.lo[r], hi = Rv.hi[r];
    int64_t c0 = lo + (int64_t)item.y * a.seg_len;
    int64_t c1 = min(hi, c0 + a.seg_len);
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(Rv.rows + (int64_t)r * Rv.n_iso * K);
    for (int i = threadIdx.x; i < Rv.n_iso * KW; i += blockDim.x) srow[i / KW][i % KW] = rw[i];  // KP == K
    __syncthreads();
    const Best t = scan_columns<K>(P, Rv, r, c0, c1, srow, sbest, a.counters);
    if (threadIdx.x == 0) a.partials[a.slot_base[r] + item.y] = to_partial(t, c1 > c0);
    __syncthreads();  // shared rows / bests are reused by the next item
  }
}

// Bulk pass for the ranges the tensor matcher handed over (TcArgs::bulk_*):
// every candidate of each listed range, its slab cut into kBulkPieces equal
// column pieces, one block per (range, piece); partial f * kBulkPieces + piece.
template <int K>
__global__ void __launch_bounds__(256) k_bulk(PoolView P, RangeView Rv, BulkArgs a) {
  constexpr int KW = K / 4;
  __shared__ uint32_t srow[8][KW];
  __shared__ Best sbest[8];
  const int64_t n_items = (int64_t)min(*a.n_bulk, (uint32_t)a.cap) * kBulkPieces;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int f = (int)(it / kBulkPieces), piece = (int)(it - (int64_t)f * kBulkPieces);
    const uint32_t r = a.list[f];
    const int64_t lo = Rv.lo[r], hi = Rv.hi[r];
    const int64_t len = cdiv(hi - lo, (int64_t)kBulkPieces);
    const int64_t c0 = min(hi, lo + piece * len), c1 = min(hi, c0 + len);
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(Rv.rows + (int64_t)r * Rv.n_iso * K);
    for (int i = threadIdx.x; i < Rv.n_iso * KW; i += blockDim.x) srow[i / KW][i % KW] = rw[i];
    __syncthreads();
    const Best t = scan_columns<K>(P, Rv, r, c0, c1, srow, sbest, a.counters);
    if (threadIdx.x == 0) a.partials[it] = to_partial(t, c1 > c0);
    __syncthreads();
  }
}

void launch_bulk(const PoolView& P, const RangeView& Rv, const BulkArgs& a, cudaStream_t s) {
  if (a.cap == 0) return;
  const unsigned grid = 148 * 8;  // grid-stride over the device-side item count
  if (Rv.K == 64)
    k_bulk<64><<<grid, 256, 0, s>>>(P, Rv, a);
  else if (Rv.K == 16)
    k_bulk<16><<<grid, 256, 0, s>>>(P, Rv, a);
  else
    invalid("bulk pass supports range_size 4 and 8");
  FIC_CHECK_LAUNCH();
}

// Generic K (any range size): rows zero-padded to KP = K rounded up to a
// multiple of 4 on both sides, so whole-word dp4a products are exact.
__global__ void __launch_bounds__(256) k_exact_generic(PoolView P, RangeView Rv, ExactArgs a) {
  extern __shared__ uint32_t dyn[];
  __shared__ Best sbest[8];
  const int K = Rv.K, KP = Rv.KP, KW = KP / 4;
  int64_t n_items = a.n_items;
  const uint32_t* elist = a.elist;
  if (a.plan) {  // device-side work count (n_items is then a bound)
    n_items = a.plan->n_eitems;
    elist = a.elist + a.plan->eb;
  }
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
  int2 item = a.items[it];
  uint32_t r = elist[item.x];
  int64_t lo = Rv.lo[r], hi = Rv.hi[r];
  int64_t c0 = lo + (int64_t)item.y * a.seg_len;
  int64_t c1 = min(hi, c0 + a.seg_len);
  const int n_iso = Rv.n_iso;
  const uint32_t* rw = reinterpret_cast<const uint32_t*>(Rv.rows + (int64_t)r * n_iso * KP);
  for (int i = threadIdx.x; i < n_iso * KW; i += blockDim.x) dyn[i] = rw[i];
  __syncthreads();
  const RangeInfo inf = Rv.info[r];
  const double n = (double)K;
  Best b;
  best_init(b);
  unsigned long long evals = 0;
  for (int64_t p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
    const uint32_t* dw = reinterpret_cast<const uint32_t*>(P.src.raw + p * KP);
    uint2 sm = P.sums[p];
    double sd = (double)sm.x, sdd = (double)sm.y, inv = P.inv_den[p];
    const uint32_t dom = pool_id(P, p);
    for (int i = 0; i < n_iso; ++i) {
      uint32_t acc = 0;
      for (int q = 0; q < KW; ++q) acc = __dp4a(__ldg(dw + q), dyn[i * KW + q], acc);
      Cand c = eval_candidate((double)acc, sd, sdd, inv, inf.sr, inf.srr, n);
      b.pre = fmin(b.pre, c.pre);
      if (better(c.err, dom, i, b.err, b.dom, b.iso)) {
        b.err = c.err;
        b.dom = dom;
        b.iso = i;
        b.sq = c.sq;
        b.oq = c.oq;
      }
    }
    evals += n_iso;
  }
  for (int m = 16; m >= 1; m >>= 1) best_merge(b, shfl_best(b, m));
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sbest[warp] = b;
  for (int m = 16; m >= 1; m >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, m);
  if (lane == 0 && evals) atomicAdd(a.counters, evals);
  __syncthreads();
  if (threadIdx.x == 0) {
    Best t = sbest[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best_merge(t, sbest[w]);
    Partial out;
    out.err = t.err;
    out.pre = t.pre;
    out.dom = t.dom;
    out.iso = (uint8_t)t.iso;
    out.sq = (uint8_t)t.sq;
    out.oq = (uint8_t)t.oq;
    out.valid = (c1 > c0) ? 1 : 0;
    a.partials[a.slot_base[r] + item.y] = out;
  }
  __syncthreads();  // shared rows / bests are reused by the next item
  }
}

void launch_exact(const PoolView& P, const RangeView& Rv, const ExactArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  // one block per item; with a device-side count, a grid-stride loop over
  // at most 4 blocks per SM
  unsigned grid = (unsigned)(a.plan ? std::min<int64_t>(a.n_items, 148 * 4) : a.n_items);
  if (Rv.K == 64)
    k_exact<64><<<grid, 256, 0, s>>>(P, Rv, a);
  else if (Rv.K == 16)
    k_exact<16><<<grid, 256, 0, s>>>(P, Rv, a);
  else
    k_exact_generic<<<grid, 256, (size_t)Rv.n_iso * Rv.KP, s>>>(P, Rv, a);
  FIC_CHECK_LAUNCH();
}

// K6: merge partials (per range) into the raster-order outputs.
__global__ void k_merge(MergeArgs a) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.R) return;
  int ns = a.nslots[r];
  if (ns == 0) return;
  const Partial* p = a.partials + a.slot_base[r];
  // a range the bulk pass took over also has its kBulkPieces partials there
  const uint32_t bi = a.bulk_idx ? a.bulk_idx[r] : 0u;
  const Partial* pb = bi ? a.bulk_part + (int64_t)(bi - 1) * kBulkPieces : nullptr;
  double err = INFINITY, pre = INFINITY;
  uint32_t dom = 0xffffffffu;
  int iso = 0, sq = 0, oq = 0;
  for (int i = 0; i < ns + (pb ? kBulkPieces : 0); ++i) {
    Partial q = i < ns ? p[i] : pb[i - ns];
    if (!q.valid) continue;
    pre = fmin(pre, q.pre);
    if (better(q.err, q.dom, q.iso, err, dom, iso)) {
      err = q.err;
      dom = q.dom;
      iso = q.iso;
      sq = q.sq;
      oq = q.oq;
    }
  }
  uint8_t* rec = a.records + (int64_t)r * 7;
  rec[0] = dom & 255;
  rec[1] = (dom >> 8) & 255;
  rec[2] = (dom >> 16) & 255;
  rec[3] = dom >> 24;
  rec[4] = (uint8_t)iso;
  rec[5] = (uint8_t)sq;
  rec[6] = (uint8_t)oq;
  // codec.py:263-264
  a.post_rms[r] = __dsqrt_rn(__ddiv_rn(fmax(err, 0.0), a.n));
  a.pre_rms[r] = __dsqrt_rn(__ddiv_rn(fmax(pre, 0.0), a.n));
}

void launch_merge(const MergeArgs& a, cudaStream_t s) {
  if (a.R == 0) return;
  k_merge<<<(unsigned)cdiv(a.R, 256), 256, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
}

}  // namespace fic
