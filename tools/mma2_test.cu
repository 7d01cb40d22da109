// Layout probe for tcgen05.mma.cta_group::2 (M=256, N=128, K=64, SS, SW128 K-major).
// Each CTA of a 2-CTA cluster writes its 128 A rows and its 64-row B share
// (rows 64*rank ..) into smem, the leader issues the MMA, both CTAs read their
// TMEM accumulators and write D to global; the host checks against a CPU GEMM.
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ float aval(int r, int k) { return (float)(((r * 7 + k * 3) % 11) - 5); }
__device__ __forceinline__ float bval(int n, int k) { return (float)(((n * 5 + k) % 9) - 4); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(float* D, const __grid_constant__ CUtensorMap tm, int use_tma) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;            // 128 x 128 B
  uint8_t* sB = sm + 16384;    // 64 x 128 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t holder;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int u = threadIdx.x; u < 128 * 8; u += 128) {
    int r = u / 8, c = u % 8;
    __half h[8];
    for (int e = 0; e < 8; ++e) h[e] = __float2half(aval(r + 128 * rank, c * 8 + e));
    *(uint4*)(sA + r * 128 + ((c ^ (r & 7)) << 4)) = *(uint4*)h;
  }
  __shared__ __align__(8) uint64_t fullb;
  for (int u = threadIdx.x; u < (use_tma ? 0 : 64 * 8); u += 128) {
    int r = u / 8, c = u % 8;
    __half h[8];
    for (int e = 0; e < 8; ++e) h[e] = __float2half(bval(r + 64 * rank, c * 8 + e));
    *(uint4*)(sB + r * 128 + ((c ^ (r & 7)) << 4)) = *(uint4*)h;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fullb)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tbase = holder;
  if (use_tma && threadIdx.x == 0) {
    uint32_t fb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(fb) : "r"(smem_u32(&fullb)), "r"(0));
    if (rank == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&fullb)), "r"(16384));
    asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(smem_u32(sB)), "l"((uint64_t)&tm), "r"(fb), "r"(0), "r"(64 * (int)rank) : "memory");
  }
  if (use_tma && rank == 0 && threadIdx.x == 0) {
    uint32_t ok2 = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok2) : "r"(smem_u32(&fullb)), "r"(0));
    } while (!ok2);
  }
  const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (rank == 0 && warp == 0 && lane == 0) {
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t ad = smem_desc(smem_u32(sA) + 32 * kk), bd = smem_desc(smem_u32(sB) + 32 * kk);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(kk));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
  }
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0));
  } while (!ok);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(tbase + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int row = 128 * rank + 32 * warp + lane;
    for (int e = 0; e < 32; ++e) D[row * 128 + c0 + e] = __uint_as_float(r[e]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                       const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  std::vector<__half> hb(128 * 64);
  for (int n = 0; n < 128; ++n) for (int kk = 0; kk < 64; ++kk) hb[n * 64 + kk] = __float2half((float)(((n * 5 + kk) % 9) - 4));
  __half* db; cudaMalloc(&db, hb.size() * 2); cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, 128}; cuuint64_t str[1] = {128}; cuuint32_t box[2] = {64, 64}; cuuint32_t es[2] = {1, 1};
  ((PFN)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, db, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int use_tma = 0; use_tma < 2; ++use_tma) {
  printf("use_tma=%d\n", use_tma);
  float* d;
  cudaMalloc(&d, 256 * 128 * 4);
  cudaMemset(d, 0, 256 * 128 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 16384 + 8192);
  k<<<2, 128, 1024 + 16384 + 8192>>>(d, tm, use_tma);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> h(256 * 128);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  auto av = [](int r, int k) { return (float)(((r * 7 + k * 3) % 11) - 5); };
  auto bv = [](int n, int k) { return (float)(((n * 5 + k) % 9) - 4); };
  int bad = 0;
  for (int r = 0; r < 256; ++r)
    for (int n = 0; n < 128; ++n) {
      float ref = 0;
      for (int kk = 0; kk < 64; ++kk) ref += av(r, kk) * bv(n, kk);
      if (h[r * 128 + n] != ref) {
        if (bad < 8) {
          // which n' matches?
          int match = -1;
          for (int m = 0; m < 128; ++m) {
            float rr = 0;
            for (int kk = 0; kk < 64; ++kk) rr += av(r, kk) * bv(m, kk);
            if (rr == h[r * 128 + n]) { match = m; break; }
          }
          printf("mismatch r=%d n=%d got %g ref %g (matches column %d)\n", r, n, h[r * 128 + n], ref, match);
        }
        ++bad;
      }
    }
  printf("bad = %d of %d\n", bad, 256 * 128);
  }
  return 0;
}
