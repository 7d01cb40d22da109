// Per-iteration cost of the MMA-issuer loop's building blocks (one warp per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/loop_bench tools/loop_bench.cu
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
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 %%rx;\n .reg .pred %%px;\n elect.sync %%rx|%%px, %1;\n selp.b32 %0, 1, 0, %%px;\n}\n"
      : "=r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

template <int mode>
__global__ void __launch_bounds__(640, 1) k(int iters, int nacc, int nwarps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bars[8];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 65536) / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < 8; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = holder;
  const uint32_t idesc = (1u << 4) | ((uint32_t)((mode >= 16 ? 128 : 256) >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // two issuing warps (nwarps == 2): warp 1 + w takes iterations j % 2 == w
  const uint64_t adesc = smem_desc(smem_u32(base)), bdesc = smem_desc(smem_u32(base + 16384));
  const uint32_t bar0 = smem_u32(&bars[0]);
  unsigned long long sink = 0;
  long long t0 = clock64();
  if (warp >= 1 && warp < 1 + nwarps) {
    int s = 0;
    const bool split = mode >= 16 && nwarps > 1;
    for (int j = split ? warp - 1 : 0; j < iters; j += split ? nwarps : 1) {
      switch (mode) {
        case 0: asm volatile("" ::: "memory"); break;
        case 1: __syncwarp(); break;
        case 2: sink += (unsigned)(j % nacc); break;
        case 3: sink += smem_u32(&bars[j & 7]); break;
        case 4: sink += elect_one(); break;
        case 5: asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); break;
        case 6:
          if (elect_one())
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 8 * s));
          __syncwarp();
          break;
        case 7:
        case 8:
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                           ::"r"(tbase + 256 * s), "l"(adesc + 2 * kk), "l"(bdesc + 2 * kk + (uint64_t)(s * 2048)), "r"(idesc), "r"(kk));
            if (mode == 8)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 8 * s));
          }
          __syncwarp();
          break;
        case 9:
          if (lane == 0) asm volatile("" ::: "memory");
          __syncwarp();
          break;
        case 10: asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); break;
        case 11: asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); break;
        case 12:  // screener release: fence, syncwarp, arrive on a count-1 barrier re-armed each phase
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar0 + 8 * (warp & 7)) : "memory");
          break;
        case 13: {  // tcgen05.ld x32 + wait
          uint32_t r[32];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                       : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                       : "r"(tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 32 * ((warp >> 2) & 3) + 128 * s));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          uint32_t x = 0;
#pragma unroll
          for (int e = 0; e < 32; ++e) x ^= r[e];
          sink += x;
          break;
        }
        case 14: sink += clock64(); break;
        case 20: {  // 2 waits + 8 MMA N128 (two tiles) + 3 commits
          uint32_t ok = 0;
          do {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"(bar0 + 48), "r"(1u) : "memory");
          } while (!ok);
          do {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"(bar0 + 40), "r"(1u) : "memory");
          } while (!ok);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                           ::"r"(tbase + 128 * ((2 * j + kk / 4) & 3)), "l"(adesc + 2 * (kk & 3)), "l"(bdesc + 2 * (kk & 3) + (uint64_t)(s * 1024)), "r"(idesc), "r"(kk & 3));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 8 * (j & 3)));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 32));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 32));
          }
          __syncwarp();
          break;
        }
        case 24: {  // 4 MMA N128 with the two (completed) waits interleaved after MMAs 2 and 3, 2 commits
          const bool leader = elect_one();
          auto mma = [&](int kk) {
            if (leader)
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                           ::"r"(tbase + 128 * (j & 3)), "l"(adesc + 2 * kk), "l"(bdesc + 2 * kk + (uint64_t)(s * 1024)), "r"(idesc), "r"(kk));
          };
          auto wt = [&](uint32_t b) {
            uint32_t ok = 0;
            do {
              asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                           : "=r"(ok) : "r"(b), "r"(1u) : "memory");
            } while (!ok);
          };
          mma(0);
          mma(1);
          wt(bar0 + 48);
          mma(2);
          wt(bar0 + 40);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          mma(3);
          if (leader) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 8 * (j & 3)));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 32));
          }
          __syncwarp();
          break;
        }
        case 21:
        case 22:
        case 23: {  // clock spin of 100 / 200 / 300 cycles + 4 MMA N128 + 2 commits
          const long long c0 = clock64();
          while (clock64() - c0 < 100 * (mode - 20)) {}
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                           ::"r"(tbase + 128 * (j & 3)), "l"(adesc + 2 * kk), "l"(bdesc + 2 * kk + (uint64_t)(s * 1024)), "r"(idesc), "r"(kk));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 8 * (j & 3)));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 32));
          }
          __syncwarp();
          break;
        }
        case 16:
        case 17:
        case 18:
        case 19:
          // N=128: 16 no commit, 17 one commit, 18 two commits, 19 two commits + two completed waits
          if (mode == 19) {
            uint32_t ok = 0;
            do {
              asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                           : "=r"(ok) : "r"(bar0 + 48), "r"(1u) : "memory");
            } while (!ok);
            do {
              asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                           : "=r"(ok) : "r"(bar0 + 40), "r"(1u) : "memory");
            } while (!ok);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                           ::"r"(tbase + 128 * (j & 3)), "l"(adesc + 2 * kk), "l"(bdesc + 2 * kk + (uint64_t)(s * 1024)), "r"(idesc), "r"(kk));
            if (mode >= 17)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 8 * (j & 3)));
            if (mode >= 18)
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 32));
          }
          __syncwarp();
          break;
        case 15: {  // shared-memory volatile load (threshold read)
          sink += *(volatile unsigned long long*)(base + 8 * lane);
          break;
        }
      }
      if (++s == 2) s = 0;
    }
    if (((mode >= 6 && mode <= 8) || mode >= 16) && warp == 1) {
      if (elect_one())
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 56));
      __syncwarp();
      uint32_t ok = 0;
      do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(bar0 + 56), "r"(0u) : "memory");
      } while (!ok);
    }
  }
  long long t1 = clock64();
  if (lane == 0 && warp >= 1 && warp < 1 + nwarps) atomicMax(out, (unsigned long long)(t1 - t0));
  if (sink == 12345) out[1] = sink;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main(int argc, char** argv) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int smem = 1024 + 16384 + 65536;
  const int iters = 4000;
  const char* names[] = {"empty", "syncwarp", "j % nacc", "smem addr", "elect", "tc fence after", "commit", "4 MMA N256",
                         "4 MMA N256 + commit", "lane0 branch + syncwarp", "wait::ld (none)", "tc fence before",
                         "fence+syncwarp+arrive", "tcgen05.ld x32 + wait", "clock64", "lds volatile",
                         "4 MMA N128", "4 MMA N128 + commit", "4 MMA N128 + 2 commits", "2 waits + 4 MMA N128 + 2 commits",
                         "2 waits + 8 MMA N128 + 3 commits", "spin100 + 4 MMA + 2 commits", "spin200 + 4 MMA + 2 commits",
                         "spin300 + 4 MMA + 2 commits", "4 MMA, waits interleaved, 2 commits"};
  void (*fns[])(int, int, int, unsigned long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>,
                                                      k<8>, k<9>, k<10>, k<11>, k<12>, k<13>, k<14>, k<15>,
                                                      k<16>, k<17>, k<18>, k<19>, k<20>, k<21>, k<22>, k<23>, k<24>};
  for (int nw : {1, 2}) {
    for (int mode = 6; mode < 25; ++mode) {
      if (mode > 8 && mode < 16) continue;
      if (nw == 2 && mode < 19) continue;
      cudaFuncSetAttribute(fns[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 16);
        fns[mode]<<<148, 640, smem>>>(iters, 2, nw, d);
        cudaDeviceSynchronize();
      }
      unsigned long long cyc;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      printf("nw=%2d %-26s %8.1f cycles/iter (%s)\n", nw, names[mode], (double)cyc / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
