// Microbenchmark: does tcgen05.mma (M128 N256 K16, SS operands) overlap with
// tcgen05.ld traffic from other warps, and with TMA-like smem writes?
// Modes: 1 = MMA only, 2 = LD only, 3 = both, 4 = MMA + smem store traffic.
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t sbo, uint32_t layout) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ uint32_t make_idesc(int n) { return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }

__global__ void __launch_bounds__(384, 1) k(int mode, int iters, unsigned long long* out, float* sink, int nmma, int ncols) {
  const uint32_t IDESC = make_idesc(ncols);
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 32768 * 2) / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tbase = holder;
  long long t0 = clock64();
  float acc = 0.f;
  if (warp == 1 && (mode & 1)) {
    if (lane == 0) {
      uint32_t a = smem_u32(base), b = smem_u32(base + 16384);
      uint32_t ph = 0;
      for (int i = 0; i < iters; ++i) {
        for (int kk = 0; kk < nmma; ++kk) {
          uint64_t ad = smem_desc(a + (kk & 3) * 32, 1024, 2), bd = smem_desc(b + (i & 1) * 32768 + (kk & 3) * 32, 1024, 2);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase), "l"(ad), "l"(bd), "r"(IDESC), "r"(kk));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        if (mode & 8) {  // no wait: only commits between MMA groups
          if (i == iters - 1) {
            uint32_t ok = 0;
            do {
              asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)), "r"((uint32_t)((iters - 1) & 1)));
            } while (!ok);
          }
        } else {
        uint32_t ok = 0;
        do {
          asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(ph));
        } while (!ok);
        ph ^= 1;
        }
      }
    }
  } else if (warp >= 4 && (mode & 2)) {
    uint32_t lb = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 256 + 128 * ((warp - 4) >> 2);
    for (int i = 0; i < iters * 2; ++i) {
      uint32_t r[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(lb + (i & 3) * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      float m0 = 0, m1 = 0;
#pragma unroll
      for (int e = 0; e < 32; e += 2) { m0 = fmaxf(m0, fabsf(__uint_as_float(r[e]))); m1 = fmaxf(m1, fabsf(__uint_as_float(r[e + 1]))); }
      acc += fmaxf(m0, m1);
    }
  } else if (warp >= 4 && (mode & 4)) {
    // smem store traffic comparable to TMA fills: 32 KB per iteration per CTA
    uint4* dst = (uint4*)(base + 16384 + 65536);
    for (int i = 0; i < iters; ++i)
      for (int q = threadIdx.x - 128; q < 2048; q += 256) dst[q & 1023] = make_uint4(i, q, i, q);
  }
  long long t1 = clock64();
  if (lane == 0) atomicMax(out + (warp == 1 ? 0 : 1), (unsigned long long)(t1 - t0));
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 16);
  cudaMalloc(&sink, 148 * 384 * 4);
  int smem = 1024 + 16384 + 65536 + 16384;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int iters = 2000;
  for (int cfg = 0; cfg < 8; ++cfg) {
    int nmma = (cfg % 2 == 0) ? 4 : 16;
    int ncols = (cfg / 2) % 2 ? 128 : 256;
    int mode_run = cfg >= 4 ? 9 : 1;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 16);
      k<<<148, 384, smem>>>(mode_run, iters, d, sink, nmma, ncols);
      cudaDeviceSynchronize();
    }
    unsigned long long c[2];
    cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
    printf("%s N=%d, %d MMAs (K=16) per commit: %.1f cycles per MMA (%s)\n", mode_run == 9 ? "commit-only" : "commit+wait", ncols, nmma, (double)c[0] / iters / nmma,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
