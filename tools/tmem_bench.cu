// Microbenchmark: tcgen05.ld throughput (bytes/cycle/SM) for several shapes
// and warp counts, and tcgen05.mma M=128 N=256 K=16 issue rate.  sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NW, int SHAPE>
__global__ void k_ld(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t holder;
  int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t base = holder + ((uint32_t)(32 * (warp & 3)) << 16);
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t col = ((i * 64) + (warp >> 2) * 128) & 511;
    uint32_t r[64];
    if (SHAPE == 0) {  // 32x32b.x32: 32 regs
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(base + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      float m0 = 0, m1 = 0, m2 = 0, m3 = 0;
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        m0 = fmaxf(m0, fabsf(__uint_as_float(r[e]))); m1 = fmaxf(m1, fabsf(__uint_as_float(r[e + 1])));
        m2 = fmaxf(m2, fabsf(__uint_as_float(r[e + 2]))); m3 = fmaxf(m3, fabsf(__uint_as_float(r[e + 3])));
      }
      acc += fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
    } else if (SHAPE == 2) {  // two 32x32b.x32 in flight, one wait
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(base + col));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
                   : "r"(base + col + 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      float m0 = 0, m1 = 0, m2 = 0, m3 = 0;
#pragma unroll
      for (int e = 0; e < 64; e += 4) {
        m0 = fmaxf(m0, fabsf(__uint_as_float(r[e]))); m1 = fmaxf(m1, fabsf(__uint_as_float(r[e + 1])));
        m2 = fmaxf(m2, fabsf(__uint_as_float(r[e + 2]))); m3 = fmaxf(m3, fabsf(__uint_as_float(r[e + 3])));
      }
      acc += fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
    } else if (SHAPE == 3) {  // one 32x32b.x32, no compute (pure load + wait)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(base + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += __uint_as_float(r[0]);
    } else {  // 16x256b.x8: 32 regs (rows 2x16, 64 columns... same bytes)
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(base + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += __uint_as_float(r[e]);
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)(t1 - t0));
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}

template <int NW, int SHAPE>
void run(const char* name) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 148 * NW * 32 * 4);
  int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 8);
    k_ld<NW, SHAPE><<<148, NW * 32>>>(iters, d, sink);
    cudaDeviceSynchronize();
  }
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double bytes = (double)iters * NW * 32 * 32 * 4 * (SHAPE == 2 ? 2 : 1);  // per SM
  printf("%-28s warps=%2d  %.1f B/cycle/SM  (%llu cycles, err=%s)\n", name, NW, bytes / cyc, cyc,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<4, 0>("ld x32 + max");
  run<8, 0>("ld x32 + max");
  run<16, 0>("ld x32 + max");
  run<4, 2>("ld 2 x32 + max");
  run<8, 2>("ld 2 x32 + max");
  run<16, 2>("ld 2 x32 + max");
  run<4, 3>("ld x32 only");
  run<8, 3>("ld x32 only");
  run<16, 3>("ld x32 only");
  return 0;
}
