// Shared definitions of the B200 fractal-encoder library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>
#include <string>

#include "../../include/fic_b200.h"

namespace fic {

// ---------------------------------------------------------------------------
// error handling: thread-local message + status code (fic_last_error)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
const char* last_error();

struct Error {
  int code;
  std::string msg;
};

#define FIC_CUDA(expr)                                                        \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      throw ::fic::Error{_e == cudaErrorMemoryAllocation ? FIC_ENOMEM         \
                                                         : FIC_ECUDA,         \
                         std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    }                                                                         \
  } while (0)

extern thread_local int g_launches;  // kernels launched by the current call
// true while this thread records a CUDA graph of an encode (fic_api.cu):
// timing events are then recorded as external (timestamp) nodes
extern thread_local bool g_capturing;
inline cudaError_t record_timing_event(cudaEvent_t e, cudaStream_t s) {
  return g_capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
}
#define FIC_CHECK_LAUNCH() do { ++::fic::g_launches; FIC_CUDA(cudaGetLastError()); } while (0)

inline void invalid(const std::string& msg) { throw Error{FIC_EINVAL, msg}; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device: set it
// once per (current device, kernel, size), thread-safe (fic_api.cu).
void smem_optin(const void* func, int bytes);
template <class F>
inline void smem_optin_k(F* func, int bytes) {
  smem_optin(reinterpret_cast<const void*>(func), bytes);
}

// ---------------------------------------------------------------------------
// geometry of one encode call (blocks.py / codec.py)
// ---------------------------------------------------------------------------
struct Geo {
  int H, W;
  int rs, ds, st;   // range size, domain size, domain stride
  int npx;          // rs*rs: pixels per range == decimated domain
  int nrx, nry, R;  // ranges per row / column / total (raster, x fastest)
  int ndx, ndy;     // domain positions per row / column
  int64_t D;        // domains (raster, x fastest; blocks.py:58-72)
  int n_iso;        // 8 with isometries, else 1
};

// Per-range data, FD-sorted tile order or raster order as documented.
struct RangeInfo {
  double sr, srr;   // sum r, sum r^2 (exact)
  double V;         // srr - sr^2/npx (exact: the range's sum of squared deviations)
  int32_t rho;      // round(sr/npx): A-operand centring offset
  int32_t pad;
};

// Partial best for one (work item, range).
struct Partial {
  double err;       // best post-quantisation squared error
  double pre;       // best pre-quantisation squared error
  uint32_t dom;     // raster domain index (0xffffffff = none)
  uint8_t iso, sq, oq, valid;
};

// order-preserving bits of a double (unsigned order == numeric order,
// negatives included) and back, for atomicMin / CAS on fp64 values
__host__ __device__ __forceinline__ unsigned long long ord_bits(double x) {
  unsigned long long b;
  memcpy(&b, &x, 8);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double unord_bits(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double x;
  memcpy(&x, &b, 8);
  return x;
}

// lexicographic (err, dom, iso): codec.py:243-258
__host__ __device__ __forceinline__ bool better(double e1, uint32_t d1, int i1,
                                                double e2, uint32_t d2, int i2) {
  return e1 < e2 || (e1 == e2 && (d1 < d2 || (d1 == d2 && i1 < i2)));
}

// ---------------------------------------------------------------------------
// exact fp64 evaluation of one candidate — codec.py:218-242 op for op.
// No contraction: every op is an explicit round-to-nearest intrinsic.
// ---------------------------------------------------------------------------
struct Cand {
  double pre, err;
  int sq, oq;
};

__device__ __forceinline__ double sq_err(double s, double o, double sd, double sdd,
                                         double cross, double sr, double srr, double n) {
  // codec.py:167-181
  double w = __dmul_rn(o, sd);
  w = __dsub_rn(w, cross);
  w = __dmul_rn(w, s);
  w = __dmul_rn(w, 2.0);
  double out = __dmul_rn(s, s);
  out = __dmul_rn(out, sdd);
  out = __dadd_rn(out, w);
  w = __dmul_rn(o, o);
  w = __dmul_rn(w, n);
  out = __dadd_rn(out, w);
  w = __dmul_rn(o, __dmul_rn(2.0, sr));
  out = __dsub_rn(out, w);
  return __dadd_rn(out, srr);
}

__device__ __forceinline__ Cand eval_candidate(double cross, double sd, double sdd,
                                               double inv_den, double sr, double srr,
                                               double n) {
  Cand c;
  double work = __dmul_rn(sd, sr);
  double s = __dmul_rn(cross, n);
  s = __dsub_rn(s, work);
  s = __dmul_rn(s, inv_den);
  s = fmin(fmax(s, -1.0), 1.0);
  double o = __dmul_rn(s, sd);
  o = __dsub_rn(sr, o);
  // o / n: for n a power of two (K = 16, 64, ...) the quotient is the exact
  // scaling o * 2^-k, so the multiply gives the division's bits without its
  // long Newton sequence
  const unsigned long long nb = (unsigned long long)__double_as_longlong(n);
  if ((nb & 0x000fffffffffffffull) == 0)
    o = __dmul_rn(o, __longlong_as_double((long long)((2046ull - (nb >> 52)) << 52)));
  else
    o = __ddiv_rn(o, n);
  c.pre = sq_err(s, o, sd, sdd, cross, sr, srr, n);
  o = fmin(fmax(o, -255.0), 255.0);
  double sq = rint(__dmul_rn(__dadd_rn(s, 1.0), 15.5));
  double oq = rint(__dmul_rn(__dadd_rn(o, 255.0), 127.0 / 510.0));
  double sh = __dsub_rn(__dmul_rn(sq, 2.0 / 31.0), 1.0);
  double oh = __dsub_rn(__dmul_rn(oq, 510.0 / 127.0), 255.0);
  c.err = sq_err(sh, oh, sd, sdd, cross, sr, srr, n);
  c.sq = (int)sq;
  c.oq = (int)oq;
  return c;
}


inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
__host__ __device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// host-side isometry permutation tables: flat[perm[i][k]] == iso_i(block)[k]
// (blocks.py:113-139); inverse tables are what the encoder applies to ranges.
void iso_tables(int rs, int* perm /*8*rs*rs*/, int* inv_perm /*8*rs*rs*/);

}  // namespace fic
