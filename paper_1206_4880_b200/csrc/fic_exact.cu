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

__device__ __forceinline__ void cas128(unsigned long long* addr, unsigned long long cmp_lo,
                                       unsigned long long cmp_hi, unsigned long long new_lo,
                                       unsigned long long new_hi, unsigned long long& old_lo,
                                       unsigned long long& old_hi) {
  asm volatile(
      "{\n .reg .b128 d, b, c;\n mov.b128 b, {%2, %3};\n mov.b128 c, {%4, %5};\n"
      " atom.global.cas.b128 d, [%6], b, c;\n mov.b128 {%0, %1}, d;\n}\n"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi), "l"(addr)
      : "memory");
}

// Survivor-list rescoring (SlArgs).  A warp takes 32 entries, stages them
// and the prefix sums of their popcounts in shared memory, and deals their
// candidates (set mask bits) round-robin to its lanes, so every lane
// evaluates whatever the masks' sizes.  Each candidate goes through
// eval_candidate (the reference's fp64 sequence); improvements of the
// range's best are published with a 128-bit CAS on (ord(err), dom | iso |
// s_q | o_q), whose unsigned order is the lexicographic (err, dom, iso)
// order, and the pre-quantisation error with a 64-bit atomicMin on ord(pre).
template <int K>
__global__ void __launch_bounds__(256) k_sl_rescore(PoolView P, RangeView Rv, SlArgs a) {
  constexpr int KW = K / 4;
  __shared__ uint4 s_ent[8][32];
  __shared__ uint32_t s_incl[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n = (int64_t)min(*a.sl_count, a.sl_cap);
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n_iso = Rv.n_iso;
  const double nK = (double)K;
  unsigned long long evals = 0;
  for (int64_t base = warp0 * 32; base < n; base += nwarps * 32) {
    uint4 e = make_uint4(0, 0, 0, 0);
    if (base + lane < n) e = a.sl[base + lane];
    const unsigned long long mask = ((unsigned long long)e.w << 32) | e.z;
    uint32_t incl = (uint32_t)__popcll(mask);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    s_ent[w][lane] = e;
    s_incl[w][lane] = incl;
    __syncwarp();
    const uint32_t total = s_incl[w][31];
    for (uint32_t t = lane; t < total; t += 32) {
      int j = 0;  // first entry whose inclusive count exceeds t
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1)
        if (s_incl[w][j + step - 1] <= t) j += step;
      const uint4 ej = s_ent[w][j];
      const uint32_t k = t - (j ? s_incl[w][j - 1] : 0u);
      const uint32_t plo = (uint32_t)__popc(ej.z);
      const int bit = k < plo ? (int)__fns(ej.z, 0, (int)k + 1) : 32 + (int)__fns(ej.w, 0, (int)(k - plo) + 1);
      const int64_t p = (int64_t)ej.y + bit;
      const uint32_t rid = ej.x >> 3, iso = ej.x & 7u;
      const uint32_t dom = pool_id(P, p);
      uint32_t dw[KW];
      dom_words<K>(P, p, dom, dw);
      const uint4* rrow = reinterpret_cast<const uint4*>(Rv.rows + ((int64_t)rid * n_iso + iso) * K);
      uint32_t acc = 0;
#pragma unroll
      for (int q = 0; q < KW / 4; ++q) {
        const uint4 rv = __ldg(rrow + q);
        acc = __dp4a(dw[4 * q], rv.x, acc);
        acc = __dp4a(dw[4 * q + 1], rv.y, acc);
        acc = __dp4a(dw[4 * q + 2], rv.z, acc);
        acc = __dp4a(dw[4 * q + 3], rv.w, acc);
      }
      const uint2 sm = __ldg(P.sums + p);
      const RangeInfo inf = Rv.info[rid];
      const Cand c = eval_candidate((double)acc, (double)sm.x, (double)sm.y, __ldg(P.inv_den + p),
                                    inf.sr, inf.srr, nK);
      ++evals;
      atomicMin(a.pre + rid, ord_bits(c.pre));
      const unsigned long long khi = ord_bits(c.err);
      const unsigned long long klo = ((unsigned long long)dom << 32) | (iso << 24) |
                                     ((uint32_t)c.sq << 16) | ((uint32_t)c.oq << 8);
      unsigned long long* slot = a.best + 2 * (int64_t)rid;
      unsigned long long clo = __ldcg(slot), chi = __ldcg(slot + 1);
      while (khi < chi || (khi == chi && klo < clo)) {
        unsigned long long olo, ohi;
        cas128(slot, clo, chi, klo, khi, olo, ohi);
        if (olo == clo && ohi == chi) break;
        clo = olo;
        chi = ohi;
      }
    }
    __syncwarp();
  }
  for (int m = 16; m >= 1; m >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, m);
  if (lane == 0 && evals) atomicAdd(a.counters, evals);
}

void launch_sl_rescore(const PoolView& P, const RangeView& Rv, const SlArgs& a, cudaStream_t s) {
  if (!a.sl) return;
  const unsigned grid = 148 * 8;  // grid-stride over the device-side entry count
  if (Rv.K == 64)
    k_sl_rescore<64><<<grid, 256, 0, s>>>(P, Rv, a);
  else if (Rv.K == 16)
    k_sl_rescore<16><<<grid, 256, 0, s>>>(P, Rv, a);
  else
    invalid("survivor list supports range_size 4 and 8");
  FIC_CHECK_LAUNCH();
}

// Hit list (TcArgs::hl): one warp per entry.  Each lane holds two of the
// chunk's 64 columns (decimated words, sum_d, K den) and, for lane j < the
// number of hit rows, the j-th hit row's range data, all loaded at once.
// The rows are then taken in turn (shuffled from their lane): every column
// of the row's slab gets the exact lower bound test in integer / fp32
// arithmetic, and the candidates that can still win or tie go to a per-warp
// queue in shared memory that is evaluated 32 at a time with all lanes
// (codec.py:218-258 via eval_candidate), publishing to the survivor list's
// best / pre arrays only when a candidate beats what they hold.
#ifndef FIC_HL_BLK
#define FIC_HL_BLK 3  // resident blocks per SM (register budget) of k_hl_rescore
#endif
namespace {
constexpr int HLQ = 128;  // queue slots per warp (< 32 queued + 64 of one row)
}

template <int K>
__device__ __forceinline__ void hl_flush(const PoolView& P, const RangeView& Rv, const HlArgs& a,
                                         const uint4* q, uint32_t head, int cnt, int lane,
                                         unsigned long long& evals) {
  if (lane < cnt) {
    const uint4 c = q[(head + lane) & (HLQ - 1)];  // (rid, pool position, cross, iso)
    const uint32_t rid = c.x, iso = c.w;
    const int64_t p = c.y;
    // every load first (one round trip): column, range, and the current bests
    unsigned long long* slot = a.best + 2 * (int64_t)rid;
    const uint2 sm = __ldg(P.sums + p);
    const uint32_t did = pool_id(P, p);
    const double inv = __ldg(P.inv_den + p);
    const RangeInfo inf = Rv.info[rid];
    const unsigned long long cpre = __ldcg(a.pre + rid);
    unsigned long long clo = __ldcg(slot), chi = __ldcg(slot + 1);
    const Cand cd = eval_candidate((double)c.z, (double)sm.x, (double)sm.y, inv, inf.sr, inf.srr, (double)K);
    ++evals;
    const unsigned long long kpre = ord_bits(cd.pre);
    if (kpre < cpre) atomicMin(a.pre + rid, kpre);
    const unsigned long long khi = ord_bits(cd.err);
    const unsigned long long klo = ((unsigned long long)did << 32) | (iso << 24) |
                                   ((uint32_t)cd.sq << 16) | ((uint32_t)cd.oq << 8);
    while (khi < chi || (khi == chi && klo < clo)) {
      unsigned long long olo, ohi;
      cas128(slot, clo, chi, klo, khi, olo, ohi);
      if (olo == clo && ohi == chi) break;
      clo = olo;
      chi = ohi;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(256, FIC_HL_BLK) k_hl_rescore(PoolView P, RangeView Rv, HlArgs a) {
  constexpr int KW = K / 4;
  __shared__ uint4 s_q[8][HLQ];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint4* q = s_q[wib];
  uint32_t head = 0, tail = 0;  // queue (warp-uniform counters)
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // sorted by chunk column (k_hl_sort): each warp takes a contiguous run and
  // loads a chunk's columns once for all its entries; else a grid stride
  const uint4* L = a.sorted ? a.sorted : a.hl;
  const int64_t n = a.sorted ? (int64_t)*a.n_sorted : (int64_t)min(*a.hl_count, a.hl_cap);
  // sorted: runs of HLRUN consecutive entries handed out by an atomic
  // counter (their costs vary: a static cut leaves a tail)
  constexpr int HLRUN = 64;
  int64_t i0 = warp0, i1 = n, step = nwarps;
  if (a.sorted) {
    uint32_t r0 = 0;
    if (lane == 0) r0 = atomicAdd(a.run_ctr, 1u);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    i0 = min(n, (int64_t)r0 * HLRUN);
    i1 = min(n, i0 + HLRUN);
    step = 1;
  }
  const int iso_sh = Rv.n_iso == 8 ? 3 : 0;  // n_iso is 8 or 1 (launch_hl_rescore checks)
  const int n_iso = Rv.n_iso;
  const uint32_t* tl = a.tlist + (a.plan ? a.plan->tb : 0);
  unsigned long long evals = 0, tests = 0;
  // the current chunk's columns: lane and lane + 32 (sum_d, and K den = K (K
  // sum_dd - sum_d^2) in fp32; 0 for a flat domain)
  uint32_t cur_z = 0xffffffffu;
  uint32_t pc[2], dw[2][KW];
  int32_t sd[2];
  float kden[2];
  uint4 en = i0 < i1 ? L[i0] : make_uint4(0, 0, 0, 0);  // next entry (prefetched)
  for (int64_t i = i0; i < i1; i += step) {
    const uint4 e = en;
    if (a.sorted && i + 1 == i1) {  // next run
      uint32_t r0 = 0;
      if (lane == 0) r0 = atomicAdd(a.run_ctr, 1u);
      r0 = __shfl_sync(0xffffffffu, r0, 0);
      const int64_t n0 = min(n, (int64_t)r0 * HLRUN);
      if (n0 < n) {
        i = n0 - 1;  // the loop increment lands on n0
        i1 = min(n, n0 + HLRUN);
      }
    }
    if (i + step < i1) en = L[i + step];
    if (e.w == 0) continue;
    // lane L with bit L of the ballot loads row e.y + L: range id, isometry,
    // slab, sum_r, bound, pixels (n_iso is 1 or 8: a shift)
    uint32_t rid = 0, iso = 0;
    int32_t lo = 0, hi = 0, sr = 0;
    float cth = -1.0f;  // V - threshold - margin, rounded down (<= 0: no bound)
    uint32_t rw[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) rw[w] = 0;
    if ((e.w >> lane) & 1u) {
      const int row = (int)e.y + lane, kl = row >> iso_sh;
      iso = (uint32_t)(row - (kl << iso_sh));
      rid = __ldg(tl + e.x + kl);
      lo = Rv.lo[rid];
      hi = Rv.hi[rid];
      const RangeInfo inf = Rv.info[rid];
      sr = (int32_t)inf.sr;
      const double thr = fmin(__longlong_as_double((long long)__ldcg(a.thr_g + rid)),
                              unord_bits(__ldcg(a.best + 2 * (int64_t)rid + 1)));
      cth = __double2float_rd(inf.V - thr - 1e-5);
      const uint4* rrow = reinterpret_cast<const uint4*>(Rv.rows + ((int64_t)rid * n_iso + iso) * K);
#pragma unroll
      for (int q4 = 0; q4 < KW / 4; ++q4) {
        const uint4 v = __ldg(rrow + q4);
        rw[4 * q4] = v.x;
        rw[4 * q4 + 1] = v.y;
        rw[4 * q4 + 2] = v.z;
        rw[4 * q4 + 3] = v.w;
      }
    }
    if (e.z != cur_z) {  // warp-uniform
    cur_z = e.z;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      pc[c] = e.z + (uint32_t)(lane + 32 * c);
      sd[c] = 0;
      kden[c] = 0.0f;
#pragma unroll
      for (int w = 0; w < KW; ++w) dw[c][w] = 0;
      if ((int64_t)pc[c] < P.D) {
        dom_words<K>(P, pc[c], pool_id(P, pc[c]), dw[c]);
        const uint2 sm = __ldg(P.sums + pc[c]);
        sd[c] = (int32_t)sm.x;
        if (K == 16) {  // K sum_dd, sum_d^2 < 2^31: int32, then K den in fp32 (2^-24 rounding)
          kden[c] = (float)K * (float)((int32_t)(K * sm.y) - (int32_t)(sm.x * sm.x));
        } else {
          const long long den = (long long)K * sm.y - (long long)sm.x * sm.x;
          kden[c] = __ll2float_rn((long long)K * den);
        }
      }
    }
    }
    for (unsigned bal = e.w; bal; bal &= bal - 1) {
      const int j = __ffs(bal) - 1;  // the row's lane
      const uint32_t rj = __shfl_sync(0xffffffffu, rid, j), ij = __shfl_sync(0xffffffffu, iso, j);
      const int32_t loj = __shfl_sync(0xffffffffu, lo, j), hij = __shfl_sync(0xffffffffu, hi, j);
      const int32_t srj = __shfl_sync(0xffffffffu, sr, j);
      const float cthj = __shfl_sync(0xffffffffu, cth, j);
      uint32_t rwj[KW];
#pragma unroll
      for (int w = 0; w < KW; ++w) rwj[w] = __shfl_sync(0xffffffffu, rw[w], j);
      bool pass[2];
      uint32_t cross[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t acc = 0;
#pragma unroll
        for (int w = 0; w < KW; ++w) acc = __dp4a(dw[c][w], rwj[w], acc);
        cross[c] = acc;
        const bool in = (int32_t)pc[c] >= loj && (int32_t)pc[c] < hij;
        // every (s, o) has error >= V - num^2 / (K den) (>= V for a flat
        // domain): num = K cross - sum_r sum_d is an exact int32 (|num| <
        // 2^31 for K <= 64); the fp32 comparison keeps a 2^-18 relative
        // margin over its few roundings, so it never drops a candidate the
        // exact bound keeps
        const int32_t num = K * (int32_t)acc - srj * sd[c];
        const float nf = (float)num;
        pass[c] = in && (cthj <= 0.0f || (kden[c] > 0.0f && nf * nf >= kden[c] * cthj * (1.0f - 0x1p-18f)));
        tests += in ? 1 : 0;
      }
      // queue the passing candidates (lane order), evaluate in batches of 32
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, pass[c]);
        if (pass[c]) q[(tail + __popc(m & ((1u << lane) - 1u))) & (HLQ - 1)] = make_uint4(rj, pc[c], cross[c], ij);
        tail += (uint32_t)__popc(m);
      }
      __syncwarp();
      while (tail - head >= 32u) {
        hl_flush<K>(P, Rv, a, q, head, 32, lane, evals);
        head += 32;
        __syncwarp();
      }
    }
  }
  if (tail != head) hl_flush<K>(P, Rv, a, q, head, (int)(tail - head), lane, evals);
  for (int m = 16; m >= 1; m >>= 1) {
    evals += __shfl_xor_sync(0xffffffffu, evals, m);
    tests += __shfl_xor_sync(0xffffffffu, tests, m);
  }
  if (lane == 0 && evals) atomicAdd(a.counters, evals);
  if (lane == 0 && tests) atomicAdd(a.tests, tests);
}

// Counting sort of the hit list by chunk column (bin = column / 64), so
// k_hl_rescore can load a chunk's column data once for all of its entries
// (cfg4: ~2,600 entries per chunk from 4,096 tiles).  Order inside a bin is
// arbitrary: the per-range lexicographic minimum does not depend on it.
__global__ void k_hl_hist(const uint4* hl, const uint32_t* cnt, uint32_t cap, uint32_t* hist) {
  const int64_t n = (int64_t)min(*cnt, cap);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 e = hl[i];
    if (e.w) atomicAdd(hist + (e.z >> 6), 1u);
  }
}

// exclusive scan of nbins counts in place (one block), total to *total
__global__ void __launch_bounds__(1024) k_hl_scan(uint32_t* hist, int nbins, uint32_t* total) {
  __shared__ uint32_t s_w[32];
  const int t = threadIdx.x, per = (nbins + 1023) / 1024;
  const int b0 = min(nbins, t * per), b1 = min(nbins, b0 + per);
  uint32_t sum = 0;
  for (int b = b0; b < b1; ++b) sum += hist[b];
  uint32_t incl = sum;
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = s_w[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += v;
    }
    s_w[lane] = x;
  }
  __syncthreads();
  uint32_t run = incl - sum + (w ? s_w[w - 1] : 0u);
  for (int b = b0; b < b1; ++b) {
    const uint32_t c = hist[b];
    hist[b] = run;
    run += c;
  }
  if (t == 1023) *total = run;
}

__global__ void k_hl_scatter(const uint4* hl, const uint32_t* cnt, uint32_t cap, uint32_t* cursor,
                             uint4* out) {
  const int64_t n = (int64_t)min(*cnt, cap);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 e = hl[i];
    if (e.w) out[atomicAdd(cursor + (e.z >> 6), 1u)] = e;
  }
}

// Few bins (cfg4: 4,049 for 2,600 entries each): global atomics on one bin
// serialise, so each block counts a contiguous slice in shared memory,
// reserves its bins' ranges with one global atomic per (block, bin), and
// places its entries with shared-memory atomics.
__global__ void __launch_bounds__(512) k_hl_hist_smem(const uint4* hl, const uint32_t* cnt,
                                                      uint32_t cap, uint32_t* hist, int nbins) {
  extern __shared__ uint32_t sh[];  // [nbins]
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int64_t n = (int64_t)min(*cnt, cap);
  const int64_t per = (n + gridDim.x - 1) / gridDim.x, s0 = min(n, per * blockIdx.x), s1 = min(n, s0 + per);
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
    const uint4 e = hl[i];
    if (e.w) atomicAdd(sh + (e.z >> 6), 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, sh[b]);
}

__global__ void __launch_bounds__(512) k_hl_scatter_smem(const uint4* hl, const uint32_t* cnt,
                                                         uint32_t cap, uint32_t* cursor, uint4* out,
                                                         int nbins) {
  extern __shared__ uint32_t sh[];  // [nbins] counts -> bases
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int64_t n = (int64_t)min(*cnt, cap);
  const int64_t per = (n + gridDim.x - 1) / gridDim.x, s0 = min(n, per * blockIdx.x), s1 = min(n, s0 + per);
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
    const uint4 e = hl[i];
    if (e.w) atomicAdd(sh + (e.z >> 6), 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    if (sh[b]) sh[b] = atomicAdd(cursor + b, sh[b]);  // this block's range of bin b
  __syncthreads();
  for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
    const uint4 e = hl[i];
    if (e.w) out[atomicAdd(sh + (e.z >> 6), 1u)] = e;
  }
}

void launch_hl_sort(const HlArgs& a, int64_t D, cudaStream_t s) {
  if (!a.hl || !a.sorted) return;
  const int nbins = (int)((D + 63) / 64) + 1;
  FIC_CUDA(cudaMemsetAsync(a.bins, 0, (size_t)nbins * sizeof(uint32_t), s));
  const size_t smem = (size_t)nbins * sizeof(uint32_t);
  const bool in_smem = smem <= 96 * 1024;
  if (in_smem) {
    smem_optin_k(k_hl_hist_smem, (int)smem);
    smem_optin_k(k_hl_scatter_smem, (int)smem);
    k_hl_hist_smem<<<148 * 2, 512, smem, s>>>(a.hl, a.hl_count, a.hl_cap, a.bins, nbins);
  } else {
    k_hl_hist<<<148 * 8, 256, 0, s>>>(a.hl, a.hl_count, a.hl_cap, a.bins);
  }
  FIC_CHECK_LAUNCH();
  k_hl_scan<<<1, 1024, 0, s>>>(a.bins, nbins, const_cast<uint32_t*>(a.n_sorted));
  FIC_CHECK_LAUNCH();
  if (in_smem)
    k_hl_scatter_smem<<<148 * 2, 512, smem, s>>>(a.hl, a.hl_count, a.hl_cap, a.bins,
                                                  const_cast<uint4*>(a.sorted), nbins);
  else
    k_hl_scatter<<<148 * 8, 256, 0, s>>>(a.hl, a.hl_count, a.hl_cap, a.bins, const_cast<uint4*>(a.sorted));
  FIC_CHECK_LAUNCH();
}

void launch_hl_rescore(const PoolView& P, const RangeView& Rv, const HlArgs& a, cudaStream_t s) {
  if (!a.hl) return;
  if (Rv.n_iso != 8 && Rv.n_iso != 1) invalid("hit list needs 1 or 8 isometries");
  // one resident wave (the sorted list is cut into one contiguous run per
  // warp: a second, partial wave would leave SMs idle at the end)
  int dev = 0, sms = 148;
  FIC_CUDA(cudaGetDevice(&dev));
  FIC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)(sms * FIC_HL_BLK);
  if (Rv.K == 64)
    k_hl_rescore<64><<<grid, 256, 0, s>>>(P, Rv, a);
  else if (Rv.K == 16)
    k_hl_rescore<16><<<grid, 256, 0, s>>>(P, Rv, a);
  else
    invalid("hit list supports range_size 4 and 8");
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

// K6: merge partials (per range) into the raster-order outputs.  One warp
// per range: the lanes stride over its partial slots,
// then a lexicographic warp reduction; the survivor list's best joins in.
__global__ void k_merge(MergeArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= a.R) return;
  const int ns = a.nslots[r];
  if (ns == 0) return;
  const Partial* p = a.partials + a.slot_base[r];
  Best b;
  best_init(b);
  if (a.sl_best && lane == 0) {  // the survivor list's best for this range (k_sl_rescore)
    const unsigned long long hi = a.sl_best[2 * r + 1], lo = a.sl_best[2 * r];
    if (hi != ord_bits(INFINITY)) {
      b.err = unord_bits(hi);
      b.dom = (uint32_t)(lo >> 32);
      b.iso = (int)((lo >> 24) & 255u);
      b.sq = (int)((lo >> 16) & 255u);
      b.oq = (int)((lo >> 8) & 255u);
    }
    b.pre = unord_bits(a.sl_pre[r]);
  }
  for (int i = lane; i < ns; i += 32) {
    const Partial q = p[i];
    if (!q.valid) continue;
    Best c;
    c.err = q.err;
    c.pre = q.pre;
    c.dom = q.dom;
    c.iso = q.iso;
    c.sq = q.sq;
    c.oq = q.oq;
    best_merge(b, c);
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) best_merge(b, shfl_best(b, m));
  if (lane != 0) return;
  if (a.err_out) a.err_out[r] = (unsigned long long)__double_as_longlong(fmax(b.err, 0.0));
  uint8_t* rec = a.records + r * 7;
  rec[0] = b.dom & 255;
  rec[1] = (b.dom >> 8) & 255;
  rec[2] = (b.dom >> 16) & 255;
  rec[3] = b.dom >> 24;
  rec[4] = (uint8_t)b.iso;
  rec[5] = (uint8_t)b.sq;
  rec[6] = (uint8_t)b.oq;
  // codec.py:263-264
  a.post_rms[r] = __dsqrt_rn(__ddiv_rn(fmax(b.err, 0.0), a.n));
  a.pre_rms[r] = __dsqrt_rn(__ddiv_rn(fmax(b.pre, 0.0), a.n));
}

void launch_merge(const MergeArgs& a, cudaStream_t s) {
  if (a.R == 0) return;
  k_merge<<<(unsigned)cdiv((int64_t)a.R * 32, 256), 256, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
}

}  // namespace fic
