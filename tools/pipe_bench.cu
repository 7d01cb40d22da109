// Microbenchmark of the matcher's MMA -> TMEM screening pipeline (no TMA, static B).
// NMMA warps issue 4 x (M128 N K16) MMAs per tile into accumulator stage
// j % NACC and commit to tfull[acc]; NGRP groups of 4 screening warps
// (group g takes tiles j % NGRP == g) read the stage with tcgen05.ld x32 in
// 64-column halves, release it after the last load and reduce max|u|.
// Prints cycles per tile (MMA time: N/2 * 4 cycles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bench tools/pipe_bench.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph, bool sleep) {
  uint32_t ok = 0;
  if (sleep) {
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(bar), "r"(ph), "r"(0x100000u) : "memory");
    } while (!ok);
  } else {
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
    } while (!ok);
  }
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 %%rx;\n .reg .pred %%px;\n elect.sync %%rx|%%px, %1;\n selp.b32 %0, 1, 0, %%px;\n}\n"
      : "=r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr) : "memory");
}

// NACC stages of N columns; NGRP screening groups; LD: 0 no loads, 1 loads + max
template <int N, int NACC, int NGRP, int LD, int SLEEP, int NMMA, int PROD, int RES, int EXTRA, int KS>
__global__ void k(int tiles, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bars[16];
  __shared__ __align__(8) uint64_t pbars[16];  // full[8], empty[8] of the producer ring
  __shared__ volatile uint32_t qtail[512];
  __shared__ volatile uint32_t done;
  __shared__ unsigned long long thr_s[128];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 65536) / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x3c003c00u;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) qtail[i] = 0;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) thr_s[i] = 0x7ff0000000000000ull;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < 8; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[8 + b])), "r"(4));
    }
    for (int b = 0; b < 16; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&pbars[b])));
    done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = holder;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t tfull0 = smem_u32(&bars[0]), tempty0 = smem_u32(&bars[8]);
  const uint32_t full0 = smem_u32(&pbars[0]), empty0 = smem_u32(&pbars[8]);
  long long t0 = clock64();
  float accv = 0.f;
  if (PROD && warp == 0) {
    // producer ring of 8 stages: wait empty, arrive full (no data)
    for (int j = 0; j < tiles; ++j) {
      const int s = j & 7, ph = (j >> 3) & 1;
      wait_bar(empty0 + 8 * s, ph ^ 1, false);
      if (elect_one()) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full0 + 8 * s) : "memory");
      __syncwarp();
    }
  } else if (warp >= 1 && warp < 1 + NMMA) {
    const uint64_t adesc = smem_desc(smem_u32(base)), bdesc = smem_desc(smem_u32(base + 16384));
    for (int j = warp - 1; j < tiles; j += NMMA) {
      const int s = j % NACC, ph = (j / NACC) & 1;
      wait_bar(tempty0 + 8 * s, ph ^ 1, false);
      if (PROD) wait_bar(full0 + 8 * (j & 7), (j >> 3) & 1, false);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (elect_one()) {
        const uint64_t bs = bdesc + (uint64_t)(((j & 1) * N * 128 / 16) & 4095);
#pragma unroll
        for (int kk = 0; kk < KS; ++kk)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tbase + s * N), "l"(adesc + 2 * kk), "l"(bs + 2 * kk), "r"(idesc), "r"(kk));
        if (PROD) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty0 + 8 * (j & 7)));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tfull0 + 8 * s));
      }
      __syncwarp();
    }
  } else if (RES && (warp == 1 + NMMA || warp == 2 + NMMA)) {
    // rescorer-like polling: 8 queue tails per thread, nanosleep when idle
    const int t = threadIdx.x - 32 * (1 + NMMA);
    uint32_t hd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    while (done < 4u * NGRP) {
      int got = -1;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (got < 0 && hd[q] != qtail[(t + 64 * (q >> 2)) * 4 + (q & 3)]) { got = q; ++hd[q]; }
      if (got < 0) __nanosleep(256);
      else accv += 1.f;
    }
  } else if (warp >= 3 + NMMA && warp < 3 + NMMA + 4 * NGRP) {
    const int q = warp & 3, g = (warp - 3 - NMMA) >> 2;
    const uint32_t lb = tbase + ((uint32_t)(32 * q) << 16);
    for (int j = g; j < tiles; j += NGRP) {
      const int s = j % NACC, ph = (j / NACC) & 1;
      wait_bar(tfull0 + 8 * s, ph, SLEEP);
      asm volatile("tcgen05.fence::after_thread_sync;");
      float s_r = 1e30f;
      if (EXTRA) {
        const unsigned long long tb = thr_s[(32 * q + lane) >> 3];
        if (tb < 0x7ff0000000000000ull) s_r = sqrtf((float)__longlong_as_double((long long)tb));
      }
#pragma unroll 1
      for (int h = 0; h < N / 64; ++h) {
        uint32_t r[64];
        if (LD) {
          ld32(lb + s * N + 64 * h, r);
          ld32(lb + s * N + 64 * h + 32, r + 32);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        if (h == N / 64 - 1) {
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty0 + 8 * s) : "memory");
        }
        if (LD) {
          float m0 = 0, m1 = 0, m2 = 0, m3 = 0;
#pragma unroll
          for (int e = 0; e < 64; e += 8) {
            m0 = fmaxf(fmaxf(m0, fabsf(__uint_as_float(r[e]))), fabsf(__uint_as_float(r[e + 1])));
            m1 = fmaxf(fmaxf(m1, fabsf(__uint_as_float(r[e + 2]))), fabsf(__uint_as_float(r[e + 3])));
            m2 = fmaxf(fmaxf(m2, fabsf(__uint_as_float(r[e + 4]))), fabsf(__uint_as_float(r[e + 5])));
            m3 = fmaxf(fmaxf(m3, fabsf(__uint_as_float(r[e + 6]))), fabsf(__uint_as_float(r[e + 7])));
          }
          const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
          bool hit = mx > s_r;
          if (EXTRA) {
            const int e_lo = (lane * 7 - j * N - 64 * h), e_hi = e_lo + 100000;
            hit = hit && e_lo < 64 && e_hi > 0;
          }
          if (__any_sync(0xffffffffu, hit)) accv += 1.f;
          accv += mx;
        }
      }
    }
  }
  if (warp >= 3 + NMMA && warp < 3 + NMMA + 4 * NGRP && lane == 0) atomicAdd((uint32_t*)&done, 1u);
  long long t1 = clock64();
  if (lane == 0) atomicMax(out, (unsigned long long)(t1 - t0));
  sink[blockIdx.x * blockDim.x + threadIdx.x] = accv;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int N, int NACC, int NGRP, int LD, int SLEEP, int NMMA, int PROD = 0, int RES = 0, int EXTRA = 0, int KS = 4>
void run(int tiles, unsigned long long* d, float* sink) {
  const int smem = 1024 + 16384 + 65536;
  auto fn = k<N, NACC, NGRP, LD, SLEEP, NMMA, PROD, RES, EXTRA, KS>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int threads = 32 * (3 + NMMA + 4 * NGRP);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 16);
    fn<<<148, threads, smem>>>(tiles, d, sink);
    cudaDeviceSynchronize();
  }
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double per_tile = (double)cyc / tiles;
  printf("ksteps=%d res=%d extra=%d prod=%d N=%3d nacc=%d ngrp=%d ld=%d %s nmma=%d: %7.1f cycles/tile (MMA %4d, %3.0f%%) per 128 cols %6.1f %s\n", KS, RES, EXTRA, PROD, N, NACC,
         NGRP, LD, SLEEP ? "sleep" : "spin ", NMMA, per_tile, N * 2, 100.0 * N * 2 / per_tile, per_tile * 128 / N,
         cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 16);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int tiles = argc > 1 ? atoi(argv[1]) : 8000;
  run<128, 4, 2, 1, 1, 2, 1, 0, 1>(tiles, d, sink);
  // K = 16 (one MMA step per tile): screening groups 1 / 2 / 4, and without loads
  run<128, 4, 1, 1, 1, 2, 1, 0, 1, 1>(tiles, d, sink);
  run<128, 4, 2, 1, 1, 2, 1, 0, 1, 1>(tiles, d, sink);
  run<128, 4, 4, 1, 1, 2, 1, 0, 1, 1>(tiles, d, sink);
  run<128, 4, 2, 0, 1, 2, 1, 0, 1, 1>(tiles, d, sink);
  run<128, 4, 4, 0, 1, 2, 1, 0, 1, 1>(tiles, d, sink);
  run<64, 8, 4, 1, 1, 2, 1, 0, 1, 1>(tiles, d, sink);
  run<64, 8, 8, 1, 1, 2, 1, 0, 1, 1>(tiles, d, sink);
  return 0;
}
