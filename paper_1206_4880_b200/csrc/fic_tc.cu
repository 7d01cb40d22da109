// K4 — tcgen05 tensor-core matcher with a fused TMEM screening epilogue.
//
// One work item = 128 rows (RT ranges x n_iso isometries, FD-sorted so the
// tile's slabs form one contiguous union window) against a segment of that
// window's domain columns.  Per 256-column N-tile:
//
//   TMA (warp 0)  : B tile = 256 pool-ordered domains x K fp16, SW128 K-major
//   MMA (warp 1)  : tcgen05.mma.cta_group::1.kind::f16, M=128 N=256 K=16 steps,
//                   fp32 accumulator double-buffered in TMEM (2 x 256 cols)
//   epilogue (4-7): tcgen05.ld 32 columns at a time, |u| running max, and the
//                   exact fp64 rescoring of the rare survivors.
//
// The screen.  A row holds a = r[inv_perm[iso]] - rho (exact small integers),
// a column holds B = fp16((K d - sum_d) / sqrt(K den)), the centred unit-norm
// decimated domain.  Then u = a.B satisfies, in exact arithmetic,
//     LB = V - u^2 = min over (s, o) of sum((s d + o - r)^2)
// (V = the range's sum of squared deviations), so every candidate's
// post-quantisation error (codec.py:242) is >= LB.  With thr the best exact
// error already found for the range (any isometry), only candidates with
// |u| >= sqrt(V - thr - eta) can win or tie; |u_fp16 - u| <= eps is bounded
// rigorously (fp16 rounding of B, fp32 accumulation), so the kernel keeps
// every candidate with |u_fp| >= sqrt(V - thr - eta) - eps and rescores it
// exactly (eval_candidate: the reference's fp64 op order).  Results are
// therefore identical to evaluating every candidate exactly.
#include <cuda.h>
#include <cuda_fp16.h>

#include "match.h"

namespace fic {

namespace tc {

constexpr int BM = 128;       // rows per tile (TMEM lanes)
constexpr int BN = 256;       // columns per N-tile
constexpr int NTHREADS = 256; // 8 warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4-7 epilogue

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// SMEM matrix descriptor (K-major, swizzled): start>>4 | LBO 1 | SBO>>4 << 32 |
// version 1 << 46 | layout << 61  (layout 2 = SW128, 6 = SW32).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t sbo, uint32_t layout) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, M=128, N=256.
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int K>
struct Cfg {
  static constexpr int ROWB = K * 2;                  // bytes per fp16 row
  static constexpr uint32_t LAYOUT = (K == 64) ? 2u : 6u;  // SW128 / SW32
  static constexpr uint32_t SBO = 8 * ROWB;           // bytes per 8-row core group
  static constexpr int NST = (K == 64) ? 4 : 8;       // B pipeline stages
  static constexpr int A_BYTES = BM * ROWB;
  static constexpr int B_BYTES = BN * ROWB;
  static constexpr int SMEM = 1024 /*align slack*/ + A_BYTES + NST * B_BYTES + 256;
  static constexpr int KW = K / 4;                    // u32 words of a u8 row
};

// byte offset of 16-byte chunk `c` of row `r` in a swizzled K-major tile
template <int K>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  if (K == 64) return r * 128 + ((c ^ (r & 7)) << 4);
  return r * 32 + ((c ^ ((r >> 2) & 1)) << 4);
}

}  // namespace tc

using namespace tc;

template <int K>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_match_tc(const __grid_constant__ CUtensorMap tmB, PoolView P, RangeView Rv, TcArgs a) {
  using C = Cfg<K>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + C::NST * C::B_BYTES);
  // bars: full[NST], empty[NST], tfull[2], tempty[2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * C::NST + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto full_bar = [&](int s) { return smem_u32(bars + s); };
  auto empty_bar = [&](int s) { return smem_u32(bars + C::NST + s); };
  auto tfull_bar = [&](int b) { return smem_u32(bars + 2 * C::NST + b); };
  auto tempty_bar = [&](int b) { return smem_u32(bars + 2 * C::NST + 2 + b); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // pipeline state (each role advances its own copy identically)
  int stage = 0, ph = 0, acc = 0, acc_ph = 0;
  const int n_iso = Rv.n_iso;
  const double nK = (double)K;

  // ---- per-row epilogue state ----
  const int erow = threadIdx.x - 128;  // row owned by an epilogue thread
  uint32_t rr[C::KW];
  double sr = 0, srr = 0, V = 0, eps = 0;
  int32_t rlo = 0, rhi = 0;
  uint32_t rid = 0;
  bool rvalid = false;
  unsigned long long evals = 0, screened = 0;

  int prev_tile = -1;
  for (int64_t it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    const int2 item = a.items[it];
    const int tile = item.x;
    const int64_t wlo = a.wlo[tile], whi = a.whi[tile];
    const int64_t c0 = wlo + (int64_t)item.y * a.seg_len;
    const int64_t c1 = min(whi, c0 + a.seg_len);
    const int nt = (int)cdiv(c1 - c0, BN);

    if (tile != prev_tile) {
      // A operand: row j = (range k = j / n_iso, iso i = j % n_iso), a = rv - rho
      for (int u = threadIdx.x; u < BM * (K / 8); u += NTHREADS) {
        int j = u / (K / 8), c = u % (K / 8);
        int k = j / n_iso, i = j - k * n_iso;
        int64_t g = (int64_t)tile * a.RT + k;
        uint32_t h[4] = {0, 0, 0, 0};
        if (k < a.RT && g < a.n_tr) {
          uint32_t r = a.tlist[g];
          int rho = Rv.info[r].rho;
          const uint8_t* src = Rv.rows + ((int64_t)r * n_iso + i) * K + c * 8;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __half2 hv = __floats2half2_rn((float)((int)src[2 * e] - rho),
                                           (float)((int)src[2 * e + 1] - rho));
            h[e] = *reinterpret_cast<uint32_t*>(&hv);
          }
        }
        *reinterpret_cast<uint4*>(sA + swz<K>(j, c)) = make_uint4(h[0], h[1], h[2], h[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (erow >= 0) {
        int k = erow / n_iso;
        int64_t g = (int64_t)tile * a.RT + k;
        rvalid = (k < a.RT) && (g < a.n_tr);
        if (rvalid) {
          rid = a.tlist[g];
          RangeInfo inf = Rv.info[rid];
          sr = inf.sr;
          srr = inf.srr;
          V = inf.V;
          rlo = Rv.lo[rid];
          rhi = Rv.hi[rid];
          // ||a||^2 = sum (r - rho)^2 = srr - 2 rho sr + K rho^2 (exact)
          double an = (double)((int64_t)srr - 2 * (int64_t)inf.rho * (int64_t)sr +
                               (int64_t)K * inf.rho * inf.rho);
          eps = (0x1p-11 + 0x1p-12 + 0x1p-13) * sqrt(an) + (double)K * 510.0 * 0x1p-24 + 1e-6;
          const uint32_t* src = reinterpret_cast<const uint32_t*>(
              Rv.rows + ((int64_t)rid * n_iso + (erow - k * n_iso)) * K);
#pragma unroll
          for (int q = 0; q < C::KW; ++q) rr[q] = src[q];
        } else {
          rlo = rhi = 0;
        }
      }
      prev_tile = tile;
    }
    __syncthreads();

    if (warp == 0) {
      if (lane == 0) {
        for (int j = 0; j < nt; ++j) {
          mbar_wait(empty_bar(stage), ph ^ 1);
          mbar_expect_tx(full_bar(stage), C::B_BYTES);
          tma_load_2d(smem_u32(sB + stage * C::B_BYTES), &tmB, full_bar(stage), 0,
                      (int)(c0 + (int64_t)j * BN));
          if (++stage == C::NST) { stage = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        const uint32_t a_addr = smem_u32(sA);
        for (int j = 0; j < nt; ++j) {
          mbar_wait(tempty_bar(acc), acc_ph ^ 1);
          mbar_wait(full_bar(stage), ph);
          fence_after();
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
          const uint32_t d = tmem_base + acc * BN;
#pragma unroll
          for (int kk = 0; kk < K / 16; ++kk)
            mma_f16(d, smem_desc(a_addr + kk * 32, C::SBO, C::LAYOUT),
                    smem_desc(b_addr + kk * 32, C::SBO, C::LAYOUT), kk > 0 ? 1u : 0u);
          mma_commit(empty_bar(stage));
          mma_commit(tfull_bar(acc));
          if (++stage == C::NST) { stage = 0; ph ^= 1; }
          if (++acc == 2) { acc = 0; acc_ph ^= 1; }
        }
      }
    } else if (warp >= 4) {
      // ------------------------------ epilogue ------------------------------
      const int q = warp & 3;  // TMEM lane quarter == rows 32q..32q+31
      const int iso = erow % n_iso;
      double err = INFINITY, pre = INFINITY, thr = INFINITY;
      uint32_t dom = 0xffffffffu;
      int sq = 0, oq = 0;
      float s_r = -1.0f;  // |u| threshold; negative = every candidate survives
      for (int j = 0; j < nt; ++j) {
        mbar_wait(tfull_bar(acc), acc_ph);
        fence_after();
        const int64_t n0 = c0 + (int64_t)j * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int64_t p0 = n0 + 32 * c;
          if (p0 >= c1) break;  // warp-uniform
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN + 32 * c, v);
          tmem_wait_ld();
          const bool need = rvalid && p0 < rhi && p0 + 32 > rlo;
          float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            m0 = fmaxf(m0, fabsf(v[e]));
            m1 = fmaxf(m1, fabsf(v[e + 1]));
            m2 = fmaxf(m2, fabsf(v[e + 2]));
            m3 = fmaxf(m3, fabsf(v[e + 3]));
          }
          const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
          const bool hit = need && mx >= s_r;
          if (need) screened += 32;
          if (__any_sync(0xffffffffu, hit)) {
            uint32_t mask = 0;
            if (hit) {
              const int64_t lim_lo = max((int64_t)rlo, p0) - p0;
              const int64_t lim_hi = min(min((int64_t)rhi, c1), p0 + 32) - p0;
#pragma unroll
              for (int e = 0; e < 32; ++e)
                mask |= (fabsf(v[e]) >= s_r && e >= lim_lo && e < lim_hi) ? (1u << e) : 0u;
            }
            while (__any_sync(0xffffffffu, mask != 0)) {
              if (mask) {
                const int e = __ffs(mask) - 1;
                mask &= mask - 1;
                const int64_t p = p0 + e;
                uint32_t acc32 = 0;
                const uint4* src = reinterpret_cast<const uint4*>(P.raw + p * K);
#pragma unroll
                for (int w4 = 0; w4 < C::KW / 4; ++w4) {
                  uint4 dv = __ldg(src + w4);
                  acc32 = __dp4a(dv.x, rr[4 * w4], acc32);
                  acc32 = __dp4a(dv.y, rr[4 * w4 + 1], acc32);
                  acc32 = __dp4a(dv.z, rr[4 * w4 + 2], acc32);
                  acc32 = __dp4a(dv.w, rr[4 * w4 + 3], acc32);
                }
                const uint2 sm = __ldg(P.sums + p);
                const Cand cd = eval_candidate((double)acc32, (double)sm.x, (double)sm.y,
                                               __ldg(P.inv_den + p), sr, srr, nK);
                const uint32_t did = __ldg(P.ids + p);
                pre = fmin(pre, cd.pre);
                if (better(cd.err, did, iso, err, dom, iso)) {
                  err = cd.err;
                  dom = did;
                  sq = cd.sq;
                  oq = cd.oq;
                }
                thr = fmin(thr, cd.err);
                ++evals;
              }
            }
            // share the range's threshold across its isometry lanes
            for (int m = 1; m < n_iso; m <<= 1) thr = fmin(thr, __shfl_xor_sync(0xffffffffu, thr, m));
            const double cth = V - thr - 1e-5;
            if (cth > 0.0) {
              const double t = sqrt(cth) * (1.0 - 1e-9) - eps;
              s_r = __double2float_rd(t);
            } else {
              s_r = -1.0f;
            }
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty_bar(acc));
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
      // combine the n_iso rows of each range: lexicographic (err, dom, iso)
      int biso = iso;
      for (int m = 1; m < n_iso; m <<= 1) {
        double e2 = __shfl_xor_sync(0xffffffffu, err, m);
        double p2 = __shfl_xor_sync(0xffffffffu, pre, m);
        uint32_t d2 = __shfl_xor_sync(0xffffffffu, dom, m);
        int i2 = __shfl_xor_sync(0xffffffffu, biso, m);
        int s2 = __shfl_xor_sync(0xffffffffu, sq, m);
        int o2 = __shfl_xor_sync(0xffffffffu, oq, m);
        if (better(e2, d2, i2, err, dom, biso)) {
          err = e2;
          dom = d2;
          biso = i2;
          sq = s2;
          oq = o2;
        }
        pre = fmin(pre, p2);
      }
      if (rvalid && iso == 0) {
        Partial out;
        out.err = err;
        out.pre = pre;
        out.dom = dom;
        out.iso = (uint8_t)biso;
        out.sq = (uint8_t)sq;
        out.oq = (uint8_t)oq;
        out.valid = (dom != 0xffffffffu) ? 1 : 0;
        a.partials[a.slot_base[rid] + item.y] = out;
      }
    }
    __syncthreads();
  }

  if (erow >= 0) {
    for (int m = 16; m >= 1; m >>= 1) {
      evals += __shfl_xor_sync(0xffffffffu, evals, m);
      screened += __shfl_xor_sync(0xffffffffu, screened, m);
    }
    if (lane == 0) {
      atomicAdd(a.counters, evals);
      atomicAdd(a.counters + 1, screened);
    }
  }
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    FIC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      throw Error{FIC_ECUDA, "cuTensorMapEncodeTiled unavailable"};
    fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

bool tc_supported(int K) { return K == 64 || K == 16; }

template <int K>
static void launch_tc_k(const PoolView& P, const RangeView& Rv, const TcArgs& a, cudaStream_t s) {
  using C = Cfg<K>;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)P.D};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)K, (cuuint32_t)BN};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)P.bh, dims, strides,
                             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             K == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) throw Error{FIC_ECUDA, "cuTensorMapEncodeTiled failed"};
  static bool attr_set = false;
  if (!attr_set) {
    FIC_CUDA(cudaFuncSetAttribute(k_match_tc<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  C::SMEM));
    attr_set = true;
  }
  int dev = 0, sms = 148;
  FIC_CUDA(cudaGetDevice(&dev));
  FIC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  unsigned grid = (unsigned)std::min<int64_t>(a.n_items, sms);
  k_match_tc<K><<<grid, NTHREADS, C::SMEM, s>>>(map, P, Rv, a);
  FIC_CHECK_LAUNCH();
}

void launch_tc(const PoolView& P, const RangeView& Rv, const TcArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  if (Rv.K == 64)
    launch_tc_k<64>(P, Rv, a, s);
  else if (Rv.K == 16)
    launch_tc_k<16>(P, Rv, a, s);
  else
    invalid("tensor matcher supports range_size 4 and 8");
}

}  // namespace fic
