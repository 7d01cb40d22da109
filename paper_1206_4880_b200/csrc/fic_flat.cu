// Flat ranges: every pixel equal to c.  The reference's matcher
// (codec.py:184-264) then computes, for every candidate, cross = c * sum_d,
// s = (cross * n - sum_d * sum_r) * inv_den = 0 exactly, o = c exactly,
// best_pre = E(0, c) = 0, s_q = 16, o_q = rint((c + 255) * 127 / 510): the
// post-quantisation error depends on (c, sum_d, sum_dd) only and is the same
// for all isometries, so the winner is (min err, smallest raster domain id,
// isometry 0).  Ranges with the same c and slab share it: one reduction per
// value instead of screening a row the tensor screen cannot prune (its lower
// bound V - u^2 is 0 for every candidate).  Evaluation is eval_candidate,
// the same fp64 op sequence as every other path, so results are identical.
#include "kernels.h"
#include "match.h"

namespace fic {

__global__ void k_flat_detect(FlatArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.R) return;
  const int ry = r / a.nrx, rx = r - ry * a.nrx;
  const uint8_t* base = a.img + (int64_t)ry * a.rs * a.W + (int64_t)rx * a.rs;
  const int c = base[0];
  bool flat = true;
  if (a.rs == 8 && (a.W & 7) == 0) {  // aligned 8-byte rows
    const unsigned long long cc = 0x0101010101010101ull * (unsigned long long)c;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      flat = flat && (__ldg(reinterpret_cast<const unsigned long long*>(base + (int64_t)i * a.W)) == cc);
  } else {
    for (int i = 0; i < a.rs && flat; ++i)
      for (int j = 0; j < a.rs; ++j) flat = flat && (base[(int64_t)i * a.W + j] == c);
  }
  a.flat_c[r] = flat ? (int16_t)c : (int16_t)-1;
  if (flat) {
    atomicAdd(a.n_flat, 1ull);
    atomicMin(a.canon, (uint32_t)r);
  }
}

void launch_flat_detect(const FlatArgs& a, cudaStream_t s) {
  if (a.R == 0) return;
  k_flat_detect<<<(unsigned)cdiv(a.R, 256), 256, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
}

__device__ __forceinline__ bool flat_member(const FlatArgs& a, int r) {
  const uint32_t cr = *a.canon;
  return a.flat_c[r] >= 0 && a.nslots[r] > 0 && a.lo[r] == a.lo[cr] && a.hi[r] == a.hi[cr];
}

__global__ void k_flat_present(FlatArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < a.R && flat_member(a, r)) a.present[a.flat_c[r]] = 1;
}

__device__ __forceinline__ bool flat_better(const FlatArgs::Best& x, const FlatArgs::Best& y) {
  return x.err < y.err || (x.err == y.err && x.dom < y.dom);
}

constexpr int FLAT_CHUNK = 4096;

// persistent blocks over (value, chunk of the canonical slab) units
__global__ void __launch_bounds__(256) k_flat_best(PoolView P, FlatArgs a) {
  __shared__ uint8_t pres[256];
  __shared__ FlatArgs::Best red[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) pres[i] = a.present[i];
  __syncthreads();
  const uint32_t cr = *a.canon;
  const int64_t lo = a.lo[cr], hi = a.hi[cr];
  const int64_t nchunk = cdiv(hi - lo, FLAT_CHUNK);
  const double n = (double)a.K;
  for (int64_t u = blockIdx.x; u < 256 * nchunk; u += gridDim.x) {
    const int c = (int)(u / nchunk);
    const int64_t ch = u - (int64_t)c * nchunk;
    if (!pres[c]) continue;
    const double cd = (double)c, sr = n * cd, srr = n * cd * cd;
    FlatArgs::Best b{INFINITY, 0xffffffffu, 0, 0, 0};
    const int64_t p1 = min(hi, lo + (ch + 1) * FLAT_CHUNK);
    for (int64_t p = lo + ch * FLAT_CHUNK + threadIdx.x; p < p1; p += blockDim.x) {
      const uint2 sm = __ldg(P.sums + p);
      const double sd = (double)sm.x;
      const Cand q = eval_candidate(__dmul_rn(cd, sd), sd, (double)sm.y, __ldg(P.inv_den + p), sr,
                                    srr, n);
      const FlatArgs::Best x{q.err, pool_id(P, p), q.sq, q.oq, 0};
      if (flat_better(x, b)) b = x;
    }
    red[threadIdx.x] = b;
    __syncthreads();
    for (int m = blockDim.x / 2; m > 0; m >>= 1) {
      if ((int)threadIdx.x < m && flat_better(red[threadIdx.x + m], red[threadIdx.x]))
        red[threadIdx.x] = red[threadIdx.x + m];
      __syncthreads();
    }
    if (threadIdx.x == 0) a.part[(int64_t)c * a.nchunk + ch] = red[0];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_flat_reduce(FlatArgs a) {
  const int c = blockIdx.x;
  if (!a.present[c]) return;
  __shared__ FlatArgs::Best red[256];
  const uint32_t cr = *a.canon;
  const int64_t nchunk = cdiv((int64_t)a.hi[cr] - a.lo[cr], FLAT_CHUNK);
  FlatArgs::Best b{INFINITY, 0xffffffffu, 0, 0, 0};
  for (int64_t ch = threadIdx.x; ch < nchunk; ch += blockDim.x) {
    const FlatArgs::Best x = a.part[(int64_t)c * a.nchunk + ch];
    if (flat_better(x, b)) b = x;
  }
  red[threadIdx.x] = b;
  __syncthreads();
  for (int m = blockDim.x / 2; m > 0; m >>= 1) {
    if ((int)threadIdx.x < m && flat_better(red[threadIdx.x + m], red[threadIdx.x]))
      red[threadIdx.x] = red[threadIdx.x + m];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.best[c] = red[0];
}

// records and RMS of the flat ranges (as k_merge: codec.py:259-264, 399-405);
// best_pre is 0 for every candidate of a flat range
__global__ void k_flat_final(FlatArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.R || !flat_member(a, r)) return;
  const FlatArgs::Best b = a.best[a.flat_c[r]];
  uint8_t* rec = a.records + (int64_t)r * 7;
  rec[0] = b.dom & 255;
  rec[1] = (b.dom >> 8) & 255;
  rec[2] = (b.dom >> 16) & 255;
  rec[3] = b.dom >> 24;
  rec[4] = 0;
  rec[5] = (uint8_t)b.sq;
  rec[6] = (uint8_t)b.oq;
  a.post_rms[r] = __dsqrt_rn(__ddiv_rn(fmax(b.err, 0.0), (double)a.K));
  a.pre_rms[r] = 0.0;
}

void launch_flat_match(const PoolView& P, const FlatArgs& a, cudaStream_t s) {
  const unsigned rb = (unsigned)cdiv(a.R, 256);
  FIC_CUDA(cudaMemsetAsync(a.present, 0, 256, s));
  k_flat_present<<<rb, 256, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
  k_flat_best<<<148 * 8, 256, 0, s>>>(P, a);
  FIC_CHECK_LAUNCH();
  k_flat_reduce<<<256, 256, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
  k_flat_final<<<rb, 256, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
}

}  // namespace fic
