// Probe: tcgen05.mma kind::f16 with an f16 accumulator (idesc D format = 0).
// How are the 128 x N f16 results laid out in TMEM (packed two per 32-bit
// column or one per column)?  A = ones-ish small ints, B = column index / 64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/f16acc_probe tools/f16acc_probe.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// A[r][k] = (r % 7) - 3 for k < 16 (so every row has a distinct small scale),
// B[n][k] = 1 if k == 0 else 0, scaled: B[n][0] = n  -> D[r][n] = A[r][0] * n
__global__ void k(uint32_t* out, int dfmt) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;          // 128 rows x 128 B (K = 64 f16, SW128)
  uint8_t* sB = sm + 16384;  // 128 rows x 128 B
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int u = threadIdx.x; u < 128 * 8; u += 128) {
    int r = u / 8, c = u % 8;
    __half ha[8], hb[8];
    for (int e = 0; e < 8; ++e) {
      int kk = c * 8 + e;
      ha[e] = __float2half(kk == 0 ? (float)((r % 7) - 3) : 0.0f);
      hb[e] = __float2half(kk == 0 ? (float)r : 0.0f);
    }
    *(uint4*)(sA + r * 128 + ((c ^ (r & 7)) << 4)) = *(uint4*)ha;
    *(uint4*)(sB + r * 128 + ((c ^ (r & 7)) << 4)) = *(uint4*)hb;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = holder;
  // zero the 256 columns first (so unwritten cells read 0)
  {
    uint32_t z[32];
    for (int e = 0; e < 32; ++e) z[e] = 0xdeadbeefu;
    for (int c0 = 0; c0 < 256; c0 += 32)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(tbase + ((uint32_t)(32 * warp) << 16) + c0), "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]), "r"(z[16]), "r"(z[17]), "r"(z[18]), "r"(z[19]), "r"(z[20]), "r"(z[21]), "r"(z[22]), "r"(z[23]), "r"(z[24]), "r"(z[25]), "r"(z[26]), "r"(z[27]), "r"(z[28]), "r"(z[29]), "r"(z[30]), "r"(z[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // D format: bits [4,6): 0 = f16, 1 = f32
  const uint32_t idesc = ((uint32_t)dfmt << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (warp == 0 && lane == 0) {
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t ad = smem_desc(smem_u32(sA) + 32 * kk), bd = smem_desc(smem_u32(sB) + 32 * kk);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0));
  } while (!ok);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(tbase + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = 32 * warp + lane;
    for (int e = 0; e < 32; ++e) out[row * 256 + c0 + e] = r[e];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 256 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 32768);
  for (int dfmt = 0; dfmt < 2; ++dfmt) {
    k<<<1, 128, 1024 + 32768>>>(d, dfmt);
    cudaError_t e = cudaDeviceSynchronize();
    printf("dfmt=%d (%s): %s\n", dfmt, dfmt ? "f32" : "f16", cudaGetErrorString(e));
    std::vector<uint32_t> h(128 * 256);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    for (int row : {1, 2, 5}) {
      printf(" row %d:", row);
      for (int c = 0; c < 10; ++c) {
        uint32_t w = h[row * 256 + c];
        __half_raw lo, hi;
        lo.x = (unsigned short)(w & 0xffff);
        hi.x = (unsigned short)(w >> 16);
        if (dfmt)
          printf(" %g", *(float*)&w);
        else
          printf(" [%g,%g]", __half2float(__half(lo)), __half2float(__half(hi)));
      }
      printf(" ... col64 %08x col127 %08x col128 %08x\n", h[row * 256 + 64], h[row * 256 + 127], h[row * 256 + 128]);
    }
  }
  return 0;
}
