// K4 — tcgen05 tensor-core matcher with a fused TMEM screening epilogue.
//
// One work item = 128 rows (RT ranges x n_iso isometries, FD-sorted so the
// tile's slabs form one contiguous union window) against a segment of that
// window's domain columns.  Per 128-column N-tile (one CTA per SM, 12 warps):
//
//   TMA (warp 0)     : B tile = 128 pool-ordered domains x K fp16, SW128
//                      K-major, NST-stage smem ring (full/empty mbarriers)
//   MMA (warp 1)     : tcgen05.mma.cta_group::1.kind::f16, M=128 N=128, K/16
//                      steps, fp32 accumulator in NACC = 4 TMEM stages
//                      (4 x 128 columns); commits to empty[stage] + tfull[acc]
//   rescorers (2-3)  : drain the per-row survivor queues, exact fp64
//                      evaluation, publish per-range thresholds
//   screeners (4-11) : 2 groups x 4 lane quarters; group g screens the stages
//                      j % 2 == g: tcgen05.ld 2 x 32 columns, |u| max, vote,
//                      release the stage as soon as its last half is loaded
//
// Measured on B200 (tools/pipe_bench.cu, tools/loop_bench.cu): reading an
// fp32 accumulator stage back (64 KB per tile) costs about as much TMEM time
// as the MMA that wrote it, so the idealised MMA + tcgen05.ld pipeline
// plateaus near 370-390 cycles per 128x128 tile (66-70% of the MMA rate);
// per-warp latency of the screening loop and the MMA warp's two barrier
// round trips per tile are what separate this kernel from that plateau.
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
#include <cstdlib>

#include "match.h"

#ifndef FIC_TC_XP
#define FIC_TC_XP 0
#endif
#ifndef FIC_TC_SL
#define FIC_TC_SL 1  // 0: compile the survivor-list append out of the screeners
#endif
#ifndef FIC_TC_PILOT
#define FIC_TC_PILOT 1  // 0: compile the pilot screening out
#endif
#ifndef FIC_TC_BAL
#define FIC_TC_BAL 0  // 1: balanced drain of the survivor queues (measured slower: DESIGN.md)
#endif
#ifndef FIC_TC_PROF
#define FIC_TC_PROF 0  // 1: cycle accounting (debug & 4 counters) in the production instantiation
#endif
#define TCLK() ((DBG || FIC_TC_PROF) ? clock64() : 0ll)

namespace fic {

namespace tc {

constexpr int BM = 128;       // rows per tile (TMEM lanes)
#ifndef FIC_TC_BN
#define FIC_TC_BN 128
#endif
constexpr int BN = FIC_TC_BN;  // columns per N-tile (one TMEM accumulator stage)
constexpr int NACC = 512 / BN;  // TMEM accumulator stages (NACC * BN = 512 columns)
#ifndef FIC_TC_NGRP
// four groups of four screening warps (20 warps, 96 registers): pays since the hit
// ring took the hit path off the screeners (cfg3 5.59 -> 5.30 ms, cfg4 16.4 -> 15.4 ms;
// with the survivor queues it was slower than two groups at 168 registers)
#define FIC_TC_NGRP 4
#endif
#ifndef FIC_TC_NSPLIT
#define FIC_TC_NSPLIT 1
#endif
constexpr int NGRP = FIC_TC_NGRP;      // screening groups; group g handles stages j with j % NGRP == g
constexpr int NSPLIT = FIC_TC_NSPLIT;  // column slices per lane quarter within a group
constexpr int NEPI = 4 * NGRP * NSPLIT;  // screening warps: groups x slices x 4 lane quarters
constexpr int NMMA = 2;       // MMA issuing warps; warp MMA0 + w issues tiles j % NMMA == w
constexpr int NRES = 1;       // rescoring warps: thread t owns rows t + RSTRIDE * h
constexpr int NSLICE = NGRP * NSPLIT;  // survivor queues per row: one per (group, slice)
constexpr int CH = 64;        // TMEM columns per screening chunk (tcgen05.ld x32 per 32)
#ifndef FIC_TC_WIDE
#define FIC_TC_WIDE 0
#endif
constexpr bool WIDE = FIC_TC_WIDE;
#ifndef FIC_TC_F16ACC
#define FIC_TC_F16ACC 0
#endif
#ifndef FIC_TC_DUMP
#define FIC_TC_DUMP 1  // 8x8 main items hand a hit row's 64 accumulator values to the rescoring warp (hit ring); 0: per-row survivor queues
#endif
#ifndef FIC_TC_DUMP_WAIT
#define FIC_TC_DUMP_WAIT 0  // 1: a screening lane without a threshold waits for the one its hit-ring slot seeds (measured: cfg3 5.28 -> 5.38 ms; without the pilot 6.23 -> 6.14)
#endif
#ifndef FIC_TC_SLOTW
#define FIC_TC_SLOTW 68  // hit-ring slot stride in 32-bit words (64 values + row, column, window)
#endif
#ifndef FIC_TC_RES_SLEEP
#define FIC_TC_RES_SLEEP 512  // ns the rescoring warp sleeps when the hit ring is empty
#endif
#ifndef FIC_TC_RES_DIRECT
#define FIC_TC_RES_DIRECT 0  // 1: a pass whose results sit in one lane skips the per-row merge staging
#endif
#ifndef FIC_TC_LEAN
#define FIC_TC_LEAN 0  // 1: experiment, 4x4 main items without the slow path (hit list only)
#endif
// f16 accumulators for the main (non-pilot) items: a whole 128-column stage is
// read back with ONE packed tcgen05.ld (64 registers, two columns each) and
// screened with packed 3-input |x| max (VHMNMX); eps widens by the f16
// roundings of the K/16 accumulation steps
constexpr bool F16ACC = FIC_TC_F16ACC;
static_assert(!F16ACC || (BN == 128 && NSPLIT == 1 && !WIDE), "f16 accumulators: one packed load per 128-column stage");  // load a whole stage before screening (needs ~170 registers)
// Parity waits are only sound if a waiter can never be two phases ahead of a
// barrier: a group must own fixed accumulator stages (NGRP divides NACC).
static_assert(NACC % NGRP == 0, "screening groups must own whole accumulator stages");
static_assert((BN / NSPLIT) % CH == 0 && CH % 32 == 0, "slices hold whole chunks of x32 loads");
constexpr int QCAP = NSLICE > 2 ? 16 : 32;  // survivor queue entries per (row, slice); the queues fit 227 KB
constexpr uint32_t SLCH = 512;  // survivor-list entries per screening-warp chunk
constexpr uint32_t HLCH = 256;  // hit-list entries per screening-warp chunk
constexpr int PK = 8;         // pilot: |u| candidates kept per row and screening group (4x4 ranges)
#ifndef FIC_TC_PK64
#define FIC_TC_PK64 2         // (8x8 ranges)
#endif
constexpr int MMA0 = 1;       // first MMA issuing warp (warp 0: TMA producer)
constexpr int RES0 = MMA0 + NMMA;  // first rescoring warp
constexpr int RSTRIDE = 32 * NRES;
constexpr int RROWS = BM / RSTRIDE;  // rows per rescoring thread
constexpr int SCR0 = RES0 + NRES;
// warps: 0 TMA (+ TMEM alloc), MMA0.. MMA issuers, RES0.. rescorers, SCR0.. screeners
constexpr int NTHREADS = 32 * (SCR0 + NEPI);
// one CTA per SM; the register file is split per SM sub-partition (warp % 4)
constexpr int MAXREG = (16384 / (32 * ((NTHREADS / 32 + 3) / 4))) & ~7;

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

// blocking wait with a suspend-time hint: the warp sleeps in the barrier
// instead of spinning through the issue slots
#ifndef FIC_TC_SLEEP
#define FIC_TC_SLEEP 0  // 1: the screeners wait on accumulator-full with a suspend-time hint (measured: no gain)
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  if (!FIC_TC_SLEEP) {
    mbar_wait(bar, parity);
    return;
  }
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(0x100000u)
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

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
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

// kind::f16 instruction descriptor: D f32 (f16d: D f16, one value per 32-bit
// TMEM column), A/B f16, both K-major, M = 128*CG, N = BN.
template <int CG>
__device__ __forceinline__ constexpr uint32_t idesc(bool f16d = false) {
  return ((f16d ? 0u : 1u) << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
}

template <int CG>
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc,
                                        uint32_t id) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}

// MMA completion -> mbarrier arrive (in both CTAs of the pair for CG == 2)
template <int CG>
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
  else
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"((uint16_t)3)
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// shared::cluster address of the same smem location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  // default semantics, as CUTLASS's ClusterBarrier::arrive(cta_id) (the
  // .release.cluster form measured several times slower here)
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <int CG>
__device__ __forceinline__ void cta_sync() {
  if constexpr (CG == 1) {
    __syncthreads();
  } else {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
  }
}

// TMA 2D load; for CG == 2 the completion goes to the leader CTA's barrier
template <int CG>
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x,
                                         int y) {
  if constexpr (CG == 1)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
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

// 128 columns of f16 accumulators (D format f16: one value per 32-bit TMEM
// column) as 64 registers, columns 2e | 2e+1 << 16 in register e
__device__ __forceinline__ void tmem_ld64p(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// pilot key of column Q: |u| with Q in the low 6 mantissa bits, one LOP3
// ((v & km) | Q with km = 0x7FFFFFC0 in a register, Q an immediate)
template <int Q>
__device__ __forceinline__ float pilot_key(float v, uint32_t km) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(d) : "r"(__float_as_uint(v)), "n"(Q), "r"(km));
  return __uint_as_float(d);
}
// the largest key of a 64-column chunk: four FMNMX3 chains (Q = 0, 8, .., 56)
template <int Q>
__device__ __forceinline__ void pilot_max(const float* v, uint32_t km, float& m0, float& m1, float& m2,
                                          float& m3) {
  if constexpr (Q < 64) {
    m0 = fmaxf(fmaxf(m0, pilot_key<Q>(v[Q], km)), pilot_key<Q + 1>(v[Q + 1], km));
    m1 = fmaxf(fmaxf(m1, pilot_key<Q + 2>(v[Q + 2], km)), pilot_key<Q + 3>(v[Q + 3], km));
    m2 = fmaxf(fmaxf(m2, pilot_key<Q + 4>(v[Q + 4], km)), pilot_key<Q + 5>(v[Q + 5], km));
    m3 = fmaxf(fmaxf(m3, pilot_key<Q + 6>(v[Q + 6], km)), pilot_key<Q + 7>(v[Q + 7], km));
    pilot_max<Q + 8>(v, km, m0, m1, m2, m3);
  }
}

template <int K, int CG>
struct Cfg {
  static constexpr int ROWB = K * 2;                  // bytes per fp16 row
  static constexpr uint32_t LAYOUT = (K == 64) ? 2u : 6u;  // SW128 / SW32
  static constexpr uint32_t SBO = 8 * ROWB;           // bytes per 8-row core group
  static constexpr int NST = ((K == 64) ? 8 : 12) * 128 / BN;  // B smem stages
  static constexpr int A_BYTES = BM * ROWB;
  static constexpr int B_BYTES = (BN / CG) * ROWB;       // this CTA's share of a B stage
  static constexpr int TX_BYTES = BN * ROWB;              // both shares (leader's barrier)
  static constexpr int BAR_BYTES = (2 * NST + 2 * NACC + 2) * 8;
  static constexpr int ROWS_BYTES = BM * K;               // u8 permuted range rows
  static constexpr int Q_BYTES = BM * NSLICE * QCAP * 4 + BM * NSLICE * 4 * 2 + 16;  // queues + tails/heads
  static constexpr int RS_BYTES = BM * 40 + 4096;         // rescorer row state + drain staging
  static constexpr int SMEM = 1024 /*align slack*/ + A_BYTES + NST * B_BYTES + BAR_BYTES + BM * 8 + ROWS_BYTES + Q_BYTES + RS_BYTES;
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

template <int K, int CG, bool DBG, int SRC>
__global__ void __maxnreg__(MAXREG)
    k_match_tc(const __grid_constant__ CUtensorMap tmB, PoolView P, RangeView Rv, TcArgs a) {
  using C = Cfg<K, CG>;
  // CG == 2: a cluster of two CTAs runs one M = 256 tile; CTA `crank` owns
  // tile rows 128*crank .. +127 and loads columns (BN/2)*crank .. of each B stage.
  const uint32_t crank = (CG == 2) ? cluster_rank() : 0u;
  const bool leader = crank == 0;
  const int rbase = BM * (int)crank;
  // timing experiments (FIC_TC_DEBUG) compile into a separate instantiation;
  // FIC_TC_XP (compile-time, default 0) applies the same bits to the
  // production instantiation for uninstrumented experiment builds
  const int debug = DBG ? a.debug : FIC_TC_XP;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base, derived from smem_raw so accesses stay in the shared window
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + C::NST * C::B_BYTES);
  // bars: full[NST] (leader: B data landed), empty[NST] (MMA done reading B),
  // tfull[NACC] (MMA done writing D), tempty[NACC] (leader: all screeners
  // released the accumulator stage), tmem holder
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * C::NST + 2 * NACC);
  // per-range running threshold (bits of a non-negative double)
  unsigned long long* thr_s = reinterpret_cast<unsigned long long*>(
      smem + C::A_BYTES + C::NST * C::B_BYTES + C::BAR_BYTES);
  uint8_t* sRows = reinterpret_cast<uint8_t*>(thr_s + BM);      // [BM][K] u8 rows
  uint32_t* qbuf = reinterpret_cast<uint32_t*>(sRows + C::ROWS_BYTES);  // [BM][NSLICE][QCAP]
  volatile uint32_t* qtail = qbuf + BM * NSLICE * QCAP;        // [BM][NSLICE] (screener-owned)
  volatile uint32_t* qhead = qtail + BM * NSLICE;              // [BM][NSLICE] (rescorer-owned)
  volatile uint32_t* edone = qhead + BM * NSLICE;              // screening warps done
  // hit ring (FIC_TC_DUMP, 8x8 main items; aliases the survivor queues it
  // replaces): a hit lane copies its chunk's 64 accumulator values and the
  // row / column / window of the chunk into the next of NSLOT slots -- no
  // mask, no seeding, no per-survivor push on the screening warp, whose
  // stall would hold up the whole accumulator ring -- and the rescoring warp
  // filters them against the row's freshest threshold, 32 lanes per slot
  constexpr bool DUMP = FIC_TC_DUMP && K == 64;
  // slot stride in words: CH + 5 (odd: lanes reading different slots hit distinct
  // banks, scalar stores) or CH + 4 (16-byte aligned: the copy is 17 128-bit stores)
  constexpr int NSLOT = 64, SLOTW = FIC_TC_SLOTW, SLOTB = SLOTW * 4;
  static_assert(NSLOT * SLOTB + NSLOT * 4 + 16 + BM * 16 <= BM * NSLICE * QCAP * 4, "hit ring fits the queues");
  uint8_t* ring = reinterpret_cast<uint8_t*>(qbuf);                               // [NSLOT][SLOTB]
  volatile uint32_t* ring_flag = reinterpret_cast<uint32_t*>(ring + NSLOT * SLOTB);  // [NSLOT]: ticket + 1 when filled
  volatile uint32_t* ring_ticket = ring_flag + NSLOT;                              // next ticket (screeners)
  volatile uint32_t* ring_head = ring_ticket + 1;                                  // slots consumed (rescorer)
  double* rowV = reinterpret_cast<double*>(const_cast<uint32_t*>(ring_ticket) + 4);  // [BM] V of each row
  double* rowEps = rowV + BM;                                                       // [BM] screen slack
  struct RowState { double err, pre, sr, srr; uint32_t dom; uint8_t sq, oq, iso, valid; };
  RowState* rstate = reinterpret_cast<RowState*>(
      reinterpret_cast<uint8_t*>(const_cast<uint32_t*>(edone)) + 16);  // [BM]
  // balanced drain staging (rescoring warp): per lane its inclusive pending
  // count, per (lane, owned queue) pending count and head, per lane one
  // evaluated candidate
  uint32_t* s_incl = reinterpret_cast<uint32_t*>(rstate + BM);     // [32]
  uint32_t* s_crow = s_incl + 32;                                   // [32]
  uint32_t* s_cdom = s_crow + 32;                                   // [32]
  uint32_t* s_csqoq = s_cdom + 32;                                  // [32]
  double* s_cerr = reinterpret_cast<double*>(s_csqoq + 32);         // [32]
  [[maybe_unused]] double* s_cpre = s_cerr + 32;                    // [32]
  // (balanced drain only, FIC_TC_BAL; with more than two slices they would not fit RS_BYTES)
  [[maybe_unused]] uint32_t* s_pend = reinterpret_cast<uint32_t*>(s_cpre + 32);  // [32][RROWS * NSLICE]
  [[maybe_unused]] uint32_t* s_hd = s_pend + 32 * RROWS * NSLICE;                 // [32][RROWS * NSLICE]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto full_bar = [&](int s) { return smem_u32(bars + s); };
  auto empty_bar = [&](int s) { return smem_u32(bars + C::NST + s); };
  auto tfull_bar = [&](int b) { return smem_u32(bars + 2 * C::NST + b); };
  auto tempty_bar = [&](int b) { return smem_u32(bars + 2 * C::NST + NACC + b); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), (NEPI / NGRP) * CG);  // the 4 * NSPLIT warps of the stage's group
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_holder))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_holder))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  if (warp == 0 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  fence_before();
  cta_sync<CG>();
  fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // pipeline state (each role advances its own copy identically)
  int stage = 0, ph = 0;  // producer ring position (the MMA and screening warps derive theirs from gt)
  uint32_t gt = 0;  // N-tiles this CTA processed in earlier items (stage / phase bookkeeping)
  const int n_iso = Rv.n_iso;
  const double nK = (double)K;

  // ---- row identity: rescorers own row (tid - 128); screener warp (q, h)
  // owns TMEM lanes 32q..32q+31 and the h-th 128-column half of each stage
  const bool is_res = warp >= RES0 && warp < SCR0;
  const bool is_scr = warp >= SCR0;
  const int row = is_scr ? 32 * (warp & 3) + lane : 0;
  const int group = is_scr ? ((warp - SCR0) >> 2) % NGRP : 0;  // stages j % NGRP == group
  const int slice = is_scr ? ((warp - SCR0) >> 2) / NGRP : 0;  // columns slice * BN / NSPLIT ..
  constexpr int SW = BN / NSPLIT;                               // columns per slice
  const int rk = row / n_iso;          // range within this CTA's rows (thr_s index)
  const int iso = row - rk * n_iso;
  double sr = 0, srr = 0, V = 0, eps = 0;
  int32_t rlo = 0, rhi = 0;
  uint32_t rid = 0;
  bool rvalid = false;
  bool rflat = false;  // flat range on the canonical slab: the flat kernels match it
  unsigned long long evals = 0, seed_rounds = 0, hit_rounds = 0, hit_lanes = 0;
  // survivor list: each screening warp appends into its own chunk of SLCH
  // entries [sl_pos, sl_end), refilled with one global atomic per chunk (one
  // atomic per appending warp on a single counter serialised in L2); a chunk
  // starting at or past sl_cap ends the warp's list use (the queues take the rest)
  uint32_t sl_pos = 0, sl_end = 0;
  bool sl_dead = false;
  uint32_t hl_pos = 0, hl_end = 0;  // hit list: the same per-warp chunks (HLCH entries)
  bool hl_dead = false;
  long long tw0 = 0, tw1 = 0, tw2 = 0, tw3 = 0, tw4 = 0;  // stall cycles (debug & 4)
  const long long tstart = TCLK();
  unsigned long long gt_start = 0;  // debug & 8192: per-CTA start / end (globaltimer, ns)
  if (DBG && (debug & 8192) && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_start));

  // exact rescoring of pool position p, raster id `id` (codec.py:218-258
  // via eval_candidate); the domain's pixels come from the pool builder's
  // L2-resident row segments / planes (DomSrc)
  auto exact = [&](int64_t p, uint32_t id, int erow, double esr, double esrr) -> Cand {
    uint32_t dw[C::KW];
    dom_words<K, SRC>(P, p, id, dw);
    uint32_t acc32 = 0;
    const uint4* rrow = reinterpret_cast<const uint4*>(sRows + erow * K);
#pragma unroll
    for (int w4 = 0; w4 < C::KW / 4; ++w4) {
      const uint4 rv = rrow[w4];
      acc32 = __dp4a(dw[4 * w4], rv.x, acc32);
      acc32 = __dp4a(dw[4 * w4 + 1], rv.y, acc32);
      acc32 = __dp4a(dw[4 * w4 + 2], rv.z, acc32);
      acc32 = __dp4a(dw[4 * w4 + 3], rv.w, acc32);
    }
    const uint2 sm = __ldg(P.sums + p);
    return eval_candidate((double)acc32, (double)sm.x, (double)sm.y, __ldg(P.inv_den + p), esr,
                          esrr, nK);
  };

  int prev_tile = -1;
  long long tsetup = 0, tteardown = 0, nitems = 0;
  // work items are handed out dynamically (one CTA-wide fetch per item; the
  // items are ordered segment-major, so the full-length segments go first);
  // cluster pairs walk a static stride
  // s_item[k & 1] holds the k-th item of this CTA; the (k+1)-th is fetched
  // when the k-th starts, so the TMA producer can prefetch its first B tiles
  __shared__ long long s_item[2];
  __shared__ uint32_t s_rid[BM];  // CTA-local range kl -> range id (0xffffffff: none)
  __shared__ int32_t s_rho[BM];
  if (CG == 1) {
    if (threadIdx.x == 0) s_item[0] = (long long)atomicAdd(a.item_ctr, 1ull);
    __syncthreads();
  }
  int npre = 0;        // producer: B tiles of the current item issued during the previous one
  uint32_t kitem = 0;  // items this CTA started
  // virtual items: the last n_split items are each cut into nsub column
  // pieces (own partial slots), so the grid's last wave is short
  // work counts: from the device-side plan when there is one
  int64_t n_items = a.n_items, n_tr = a.n_tr, n_split = a.n_split;
  const uint32_t* tlist = a.tlist;
  if (a.plan) {
    n_items = a.plan->n_titems;
    n_tr = a.plan->n_tr;
    n_split = a.plan->n_split;
    tlist = a.tlist + a.plan->tb;
  }
  const int64_t n_whole = n_items - n_split;
  // pilot items (TcArgs::pilot_cols): one per tile, before everything else
  const int64_t n_pilot = a.pilot_cols > 0 ? (a.plan ? a.plan->n_tt : cdiv(n_tr, a.RT)) : 0;
  // (debug & 16384: the pilot items only -- a timing split, results invalid)
  const int64_t n_virt = (debug & 16384) ? n_pilot : n_pilot + n_whole + n_split * a.nsub;
  auto item_cols = [&](int64_t v, int& tile, int& slot, int64_t& c0, int64_t& c1) {
    if (v < n_pilot) {  // pilot: the first pilot_cols columns of tile v's window, no partial slot
      tile = (int)v;
      slot = -1;
      c0 = a.wlo[tile];
      c1 = max(c0, min((int64_t)a.whi[tile], c0 + a.pilot_cols));  // (the whole window when strided)
      return;
    }
    v -= n_pilot;
    int64_t i = v;
    int sub = 0;
    if (v >= n_whole) {
      i = n_whole + (v - n_whole) / a.nsub;
      sub = (int)((v - n_whole) % a.nsub);
    }
    const int2 item = a.items[i];
    tile = item.x;
    slot = item.y * a.nsub + sub;
    const int64_t wlo = a.wlo[tile], whi = a.whi[tile];
    // segment 0 is short (a.seg0 columns): run first for every tile
    // (segment-major order), it seeds the per-range thresholds cheaply
    c0 = item.y == 0 ? wlo : wlo + a.seg0 + (int64_t)(item.y - 1) * a.seg_len;
    c1 = min(whi, item.y == 0 ? c0 + a.seg0 : c0 + a.seg_len);
    if (v >= n_whole) {
      const int64_t piece = cdiv(cdiv(c1 - c0, (int64_t)a.nsub), (int64_t)BN) * BN;
      const int64_t p0 = min(c1, c0 + sub * piece);
      c1 = min(c1, p0 + piece);
      c0 = p0;
    }
  };
  // column step of a pilot item: a fixed stride, or (pilot_stride 0) about
  // pilot_samples N-tiles spread over the window (wide windows need few)
  auto pilot_step = [&](int64_t c0, int64_t c1) -> int {
    const int64_t nt_all = cdiv(c1 - c0, (int64_t)BN);
    const int64_t st = a.pilot_stride > 0 ? a.pilot_stride : max((int64_t)1, nt_all / max(1, a.pilot_samples));
    return (int)(BN * st);
  };
  for (int64_t it = (CG == 1) ? (int64_t)s_item[0] : (int64_t)(blockIdx.x / CG); it < n_virt;
       it = (CG == 1) ? (int64_t)s_item[kitem & 1] : it + gridDim.x / CG) {
    const long long ti0 = TCLK();
    ++nitems;
    if (CG == 1 && threadIdx.x == 0) s_item[(kitem + 1) & 1] = (long long)atomicAdd(a.item_ctr, 1ull);
    int tile = 0, slot = 0;
    int64_t c0 = 0, c1 = 0;
    item_cols(it, tile, slot, c0, c1);
    // pilot items sample every pilot_stride-th N-tile of the window
    const int tstep = slot < 0 ? pilot_step(c0, c1) : BN;
    const int nt = (int)cdiv(c1 - c0, (int64_t)tstep);
    // survivors of this item: the rescoring warp's queues first (overflow to
    // the survivor list), or all to the list -- for every item (sl_all 1) or
    // after each tile's first segment, the pilot that sets the thresholds (2)
    const bool pil = slot < 0;                         // a pilot item (top-PK |u| per row, no partials)
    const bool pilot = a.sl_all == 2 && slot < a.nsub;  // no list: every survivor is rescored here
    const bool list_all = FIC_TC_SL && (a.sl_all == 1 || (a.sl_all == 2 && !pilot));

    // item setup, two dependent rounds of global loads: (1) the tile's
    // range ids and rho (CTA-local range kl = row / n_iso), (2) everything
    // indexed by them (range rows -> A operand, row info, thresholds)
    const bool new_tile = tile != prev_tile;
    if (new_tile && threadIdx.x < BM) {
      const int kl = (int)threadIdx.x, kt = kl + rbase / n_iso;
      const int64_t g = (int64_t)tile * a.RT + kt;
      uint32_t r = 0xffffffffu;
      int rho = 0;
      if (kl < BM / n_iso && kt < a.RT && g < n_tr) {
        r = __ldg(tlist + g);
        rho = Rv.info[r].rho;
      }
      s_rid[kl] = r;
      s_rho[kl] = rho;
    }
    __syncthreads();
    if (new_tile) {
      // A operand: row j = (range kl = j / n_iso, iso i = j % n_iso), a = rv - rho
      constexpr int UNITS = BM * (K / 8), ROUNDS = (UNITS + NTHREADS - 1) / NTHREADS;
#pragma unroll
      for (int q = 0; q < ROUNDS; ++q) {
        const int u = (int)threadIdx.x + q * NTHREADS;
        if (u < UNITS) {
          const int j = u / (K / 8), c = u % (K / 8);
          const int kl = j / n_iso, i = j - kl * n_iso;
          const uint32_t r = s_rid[kl];
          uint32_t h[4] = {0, 0, 0, 0};
          uint2 raw8 = make_uint2(0, 0);
          if (r != 0xffffffffu) {
            const int rho = s_rho[kl];
            raw8 = __ldg(reinterpret_cast<const uint2*>(Rv.rows + ((int64_t)r * n_iso + i) * K + c * 8));
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t w = e < 2 ? raw8.x : raw8.y;
              const int b0 = (int)((w >> (16 * (e & 1))) & 255u), b1 = (int)((w >> (16 * (e & 1) + 8)) & 255u);
              __half2 hv = __floats2half2_rn((float)(b0 - rho), (float)(b1 - rho));
              h[e] = *reinterpret_cast<uint32_t*>(&hv);
            }
          }
          *reinterpret_cast<uint4*>(sA + swz<K>(j, c)) = make_uint4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<uint2*>(sRows + j * K + c * 8) = raw8;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (is_scr) {
        rvalid = s_rid[rk] != 0xffffffffu;
        rflat = false;
        if (rvalid) {
          rid = s_rid[rk];
          RangeInfo inf = Rv.info[rid];
          sr = inf.sr;
          srr = inf.srr;
          V = inf.V;
          rlo = Rv.lo[rid];
          rhi = Rv.hi[rid];
          if (a.flat_c) {
            const uint32_t cr = *a.flat_canon;
            rflat = a.flat_c[rid] >= 0 && rlo == Rv.lo[cr] && rhi == Rv.hi[cr];
          }
          // ||a||^2 = sum (r - rho)^2 = srr - 2 rho sr + K rho^2 (exact)
          double an = (double)((int64_t)srr - 2 * (int64_t)inf.rho * (int64_t)sr +
                               (int64_t)K * inf.rho * inf.rho);
          eps = (0x1p-11 + 0x1p-12 + 0x1p-13) * sqrt(an) + (double)K * 510.0 * 0x1p-24 + 1e-6;
          // f16 accumulators: each of the K/16 steps returns an f16 neighbour of
          // its sum (|sum| <= ||a|| ||B||, one ulp = 2^-10 relative; 2^-24 below
          // the normal range), plus the final value's own rounding
          if (F16ACC) eps += (double)(K / 16 + 1) * (0x1p-10 * (1.0 + 0x1p-10) * sqrt(an) + 0x1p-24);
        } else {
          rlo = rhi = 0;
        }
        if (DUMP && group == 0 && slice == 0) {
          rowV[row] = rvalid ? V : 0.0;
          rowEps[row] = rvalid ? eps : 0.0;
        }
      }
      prev_tile = tile;
    }
    if (threadIdx.x < BM) {  // per-range thresholds: start from what other segments found
      // thr_s is indexed by the CTA-local range (row / n_iso); the peer CTA
      // of a pair holds the tile's ranges from rbase / n_iso on
      const int kl = (int)threadIdx.x;
      const uint32_t r = kl < BM / n_iso ? s_rid[kl] : 0xffffffffu;
      thr_s[threadIdx.x] = r != 0xffffffffu ? a.thr_g[r] : 0x7ff0000000000000ull;  // +inf
    }
    for (int i = threadIdx.x; i < NSLICE * BM; i += NTHREADS) {
      qtail[i] = 0;
      qhead[i] = 0;
    }
    if (threadIdx.x == 0) *edone = 0;
    if (DUMP) {
      if (threadIdx.x < NSLOT) ring_flag[threadIdx.x] = 0;
      if (threadIdx.x == 0) {
        *ring_ticket = 0;
        *ring_head = 0;
      }
    }
    cta_sync<CG>();
    tsetup += TCLK() - ti0;
    const long long ti1 = TCLK();

    if (warp == 0) {
      // TMA producer: the whole warp walks the pipeline, one lane issues
      for (int j = npre; j < nt; ++j) {
        { long long t0 = TCLK(); mbar_wait(empty_bar(stage), ph ^ 1); tw0 += TCLK() - t0; }
        if ((debug & 32) && blockIdx.x == 0 && kitem == 1 && j < 64 && lane == 0) a.dbg[j * 24] = TCLK();
        if (elect_one()) {
          if ((debug & 16) || ((debug & 1024) && (j & 1))) {
            if (leader) mbar_arrive(full_bar(stage));
          } else {
            // the leader's full barrier expects both CTAs' shares
            if (leader) mbar_expect_tx(full_bar(stage), C::TX_BYTES);
            const uint32_t fb = (CG == 2) ? map_to_rank(full_bar(stage), 0) : full_bar(stage);
            tma_load<CG>(smem_u32(sB + stage * C::B_BYTES), &tmB, fb, 0,
                         (int)(c0 + (int64_t)j * tstep + (BN / CG) * (int)crank));
          }
        }
        __syncwarp();
        if (++stage == C::NST) { stage = 0; ph ^= 1; }
      }
      // prefetch the first B tiles of the next item into the ring (stages
      // free up as this item's MMAs complete); the next item skips them
      npre = 0;
      if (CG == 1 && !(debug & 16)) {
        const int64_t nit = s_item[(kitem + 1) & 1];
        if (nit < n_virt) {
          int ntile = 0, nslot = 0;
          int64_t n0 = 0, n1 = 0;
          item_cols(nit, ntile, nslot, n0, n1);
          const int nstep = nslot < 0 ? pilot_step(n0, n1) : BN;
          const int nnt = (int)cdiv(n1 - n0, (int64_t)nstep);
          const int pre = min(nnt, C::NST / 2);
          for (int j = 0; j < pre; ++j) {
            mbar_wait(empty_bar(stage), ph ^ 1);
            if (elect_one()) {
              mbar_expect_tx(full_bar(stage), C::TX_BYTES);
              tma_load<CG>(smem_u32(sB + stage * C::B_BYTES), &tmB, full_bar(stage), 0, (int)(n0 + (int64_t)j * nstep));
            }
            __syncwarp();
            if (++stage == C::NST) { stage = 0; ph ^= 1; }
          }
          npre = pre;
        }
      }
    } else if (warp >= MMA0 && warp < MMA0 + NMMA && leader) {
      // MMA issuers: NMMA warps take turns (tile j goes to warp MMA0 + j % NMMA)
      // so the issue loop's barrier round trips (~450 cycles per tile) overlap.
      // Descriptors precomputed; per K step +32 B (= +2 in the 16-byte
      // address field), per stage +B_BYTES.  Each warp's commits track its own MMAs.
      const uint64_t adesc = smem_desc(smem_u32(sA), C::SBO, C::LAYOUT);
      const uint64_t bdesc = smem_desc(smem_u32(sB), C::SBO, C::LAYOUT);
      static_assert(C::NST % NMMA == 0 && NACC % NMMA == 0, "issuer stride must divide the rings");
      const uint32_t g0 = gt + (uint32_t)(warp - MMA0);
      int stage = (int)(g0 % C::NST), ph = (int)((g0 / C::NST) & 1);
      int acc = (int)(g0 % NACC), acc_ph = (int)((g0 / NACC) & 1);
      const uint32_t full0 = full_bar(0), empty0 = empty_bar(0), tfull0 = tfull_bar(0), tempty0 = tempty_bar(0);
      for (int j = warp - MMA0; j < nt; j += NMMA) {
        { long long t0 = TCLK(); mbar_wait(tempty0 + 8 * acc, acc_ph ^ 1); tw1 += TCLK() - t0; }
        if ((debug & 32) && blockIdx.x == 0 && kitem == 1 && j < 64 && lane == 0) a.dbg[j * 24 + 2] = TCLK();
        { long long t0 = TCLK(); mbar_wait(full0 + 8 * stage, ph); tw2 += TCLK() - t0; }
        fence_after();
        if ((debug & 32) && blockIdx.x == 0 && kitem == 1 && j < 64 && lane == 0) a.dbg[j * 24 + 1] = TCLK();
        if (elect_one()) {
          const uint32_t d = tmem_base + acc * BN;
          const uint64_t bs = bdesc + (uint64_t)((stage * C::B_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < K / 16; ++kk)
            if (!(debug & 2)) mma_f16<CG>(d, adesc + 2 * kk, bs + 2 * kk, kk > 0 ? 1u : 0u, idesc<CG>(F16ACC && !pil));
          mma_commit<CG>(empty0 + 8 * stage);
          mma_commit<CG>(tfull0 + 8 * acc);
        }
        __syncwarp();
        stage += NMMA;
        if (stage >= C::NST) { stage -= C::NST; ph ^= 1; }
        acc += NMMA;
        if (acc >= NACC) { acc -= NACC; acc_ph ^= 1; }
      }
    } else if (FIC_TC_PILOT && is_scr && pil) {
      // ------------------------------ pilot ---------------------------------
      // (8x8 ranges: the best |u| per row is already a near-final threshold,
      // keep FIC_TC_PK64; 4x4 ranges need 8)
      constexpr int PKK = (K == 64) ? FIC_TC_PK64 : PK;
      // The PKK largest chunk maxima of |u| per row over the pilot columns
      // (no survivors, no seeds), in registers: their exact errors, min over
      // the range's rows, are the range's starting threshold for the main
      // items (thr_g).
      float lv[PKK];
      uint32_t lp[PKK];
      // free entries hold distinct negative sentinels, so "the entries equal
      // to the smallest" is one entry while the list fills
#pragma unroll
      for (int k = 0; k < PKK; ++k) {
        lv[k] = -1.0f - (float)k;
        lp[k] = 0;
      }
      float kth = -(float)PKK;  // smallest key in the list (negative while it has free entries)
      const uint32_t lane_base = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
      const uint32_t tfull0 = tfull_bar(0), tempty0 = tempty_bar(0);
      const int32_t lo32 = rvalid ? (int32_t)(max((int64_t)rlo, c0) - c0) : 0;
      const int32_t hi32 = rvalid ? max(lo32, (int32_t)(min((int64_t)rhi, c1) - c0)) : 0;
      for (int j = (int)((group - (int)(gt % NGRP) + NGRP) % NGRP); j < nt; j += NGRP) {
        const uint32_t gj = gt + (uint32_t)j;
        const int acc = (int)(gj % NACC), acc_ph = (int)((gj / NACC) & 1);
        mbar_wait_sleep(tfull0 + 8 * acc, acc_ph);
        fence_after();
        float mxh[SW / CH];   // each chunk's key (-inf: no column of the row's slab)
        int32_t relh[SW / CH];
#pragma unroll
        for (int h = 0; h < SW / CH; ++h) {
          float v[CH];
#pragma unroll
          for (int c = 0; c < CH / 32; ++c)
            tmem_ld32(lane_base + acc * BN + slice * SW + CH * h + 32 * c, v + 32 * c);
          tmem_wait_ld();
          if (h == SW / CH - 1) {
            fence_before();
            __syncwarp();
            if (lane == 0) {  // (a CTA pair's stage barriers live in the leader)
              if (leader)
                mbar_arrive(tempty0 + 8 * acc);
              else
                mbar_arrive_cluster(map_to_rank(tempty0 + 8 * acc, 0));
            }
          }
          const int32_t rel = j * tstep + slice * SW + CH * h;
          const int32_t e_lo = lo32 - rel, e_hi = hi32 - rel;
          const bool in_window = (uint32_t)(e_hi - 1) < (uint32_t)(hi32 - lo32 + CH - 1);
          // the chunk's largest |u| inside the row's slab, with its column:
          // key = |u| with the column index in the low 6 mantissa bits (a
          // non-negative float, so float max = integer max on the bits); the
          // truncation (2^-17 relative) only affects which near-equal
          // candidate seeds the threshold, never soundness.  Four chains over
          // the whole chunk, masked only for chunks cut by a slab edge.
          static_assert(CH == 64, "the pilot key holds a 6-bit column index");
          const uint32_t km = 0x7FFFFFC0u;
          // (debug & 512: plain |u|, a timing split)
          auto key = [&](int q) {
            return (debug & 512) ? fabsf(v[q]) : __uint_as_float((__float_as_uint(v[q]) & km) | (uint32_t)q);
          };
          float mx;
          const bool whole = e_lo <= 0 && e_hi >= CH;
          if (whole && !(debug & 512)) {
            float m0 = 0.0f, m1 = 0.0f, m2 = 0.0f, m3 = 0.0f;
            pilot_max<0>(v, km, m0, m1, m2, m3);
            mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
          } else if (whole) {
            float m0 = 0.0f, m1 = 0.0f, m2 = 0.0f, m3 = 0.0f;
#pragma unroll
            for (int q = 0; q < CH; q += 8) {
              m0 = fmaxf(fmaxf(m0, key(q)), key(q + 1));
              m1 = fmaxf(fmaxf(m1, key(q + 2)), key(q + 3));
              m2 = fmaxf(fmaxf(m2, key(q + 4)), key(q + 5));
              m3 = fmaxf(fmaxf(m3, key(q + 6)), key(q + 7));
            }
            mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
          } else {
            mx = -1.0f;
#pragma unroll
            for (int q = 0; q < CH; ++q) mx = fmaxf(mx, (q >= e_lo && q < e_hi) ? key(q) : -1.0f);
          }
          mxh[h] = (in_window && !rflat) ? mx : -INFINITY;
          relh[h] = rel;
        }
        // keep the PKK largest chunk maxima (one candidate per chunk), after
        // the stage is released: replace the first entry equal to the
        // smallest (a bitmask and its lowest bit: independent selects, no
        // chain; equal keys are common in smooth regions), new smallest by a
        // min tree
#pragma unroll
        for (int h = 0; h < SW / CH; ++h) {
          const float mx = mxh[h];
          if (!(debug & 256) && mx > kth) {  // (debug & 256: no insertion, timing)
            const uint32_t pos = (uint32_t)(relh[h] + (int)(__float_as_uint(mx) & 63u));
            uint32_t eq = 0;
#pragma unroll
            for (int kk = 0; kk < PKK; ++kk) eq |= (lv[kk] == kth) ? (1u << kk) : 0u;
            eq &= 0u - eq;
#pragma unroll
            for (int kk = 0; kk < PKK; ++kk) {
              const bool hitk = (eq >> kk) & 1u;
              lv[kk] = hitk ? mx : lv[kk];
              lp[kk] = hitk ? pos : lp[kk];
            }
            float t[PKK];
#pragma unroll
            for (int kk = 0; kk < PKK; ++kk) t[kk] = lv[kk];
#pragma unroll
            for (int w = PKK / 2; w >= 1; w >>= 1)
#pragma unroll
              for (int kk = 0; kk < w; ++kk) t[kk] = fminf(t[kk], t[kk + w]);
            kth = t[0];
          }
        }
      }
      if (debug & 256) {  // timing split: no insertions were made; evaluate 8 in-slab columns anyway
#pragma unroll
        for (int k = 0; k < PKK; ++k) {
          lv[k] = 0.0f;
          lp[k] = (uint32_t)min(lo32 + k, max(lo32, hi32 - 1));
        }
      }
      // exact errors of the list (all evaluated, branch-free, so their
      // gathers overlap; free entries repeat the first used one); the
      // range's minimum becomes its threshold
      double tnew = INFINITY;
      int kv = -1;
#pragma unroll
      for (int k = PKK - 1; k >= 0; --k)
        if (lv[k] >= 0.0f) kv = k;
      uint32_t pfirst = lp[0];
#pragma unroll
      for (int k = 1; k < PKK; ++k) pfirst = (kv == k) ? lp[k] : pfirst;
      if (rvalid && !rflat && kv >= 0 && !(debug & 2048)) {  // (debug & 2048: not evaluated, timing)
#pragma unroll
        for (int k = 0; k < PKK; ++k) {
          const int64_t pe = c0 + (lv[k] >= 0.0f ? lp[k] : pfirst);
          tnew = fmin(tnew, fmax(exact(pe, pool_id(P, pe), row, sr, srr).err, 0.0));
        }
        evals += PKK;
      }
      for (int m = 1; m < n_iso; m <<= 1) tnew = fmin(tnew, __shfl_xor_sync(0xffffffffu, tnew, m));
      if (iso == 0 && rvalid && tnew < INFINITY) {
        const unsigned long long tb = (unsigned long long)__double_as_longlong(tnew);
        atomicMin(thr_s + rk, tb);
        atomicMin(a.thr_g + rid, tb);
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicAdd((uint32_t*)edone, 1u);
    } else if (is_scr) {
      // ------------------------------ screening ------------------------------
      // Warp (group g, quarter q) owns TMEM lanes 32q.. of the stages j with
      // j % NGRP == g, read in 64-column halves: two tcgen05.ld x32, wait,
      // |u| max over 64 columns, one vote.  The accumulator stage is released
      // as soon as its last half is in registers.  Halves whose max reaches
      // the row's threshold push their survivors (positions relative to c0)
      // to the row's queue; rescoring warps do the exact evaluation.  A row
      // without an exact error yet first evaluates its best-|u| candidate
      // itself, so its threshold is finite before any survivor is pushed.
      const uint32_t lane_base = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
      const uint32_t tfull0 = tfull_bar(0), tempty0 = tempty_bar(0);
      const int32_t lo32 = rvalid ? (int32_t)(max((int64_t)rlo, c0) - c0) : 0;
      // hi32 >= lo32 always (an empty intersection is [lo32, lo32))
      const int32_t hi32 = rvalid ? max(lo32, (int32_t)(min((int64_t)rhi, c1) - c0)) : 0;
      const int qsl = group * NSPLIT + slice;
      uint32_t* myq = qbuf + (row * NSLICE + qsl) * QCAP;
      volatile uint32_t* mytail = qtail + row * NSLICE + qsl;
      volatile uint32_t* myhead = qhead + row * NSLICE + qsl;
      uint32_t qt = 0;
      unsigned long long thr_bits = 0x7ff0000000000000ull;
      float s_r = (debug & 128) ? INFINITY : -1.0f;  // |u| threshold; negative = every candidate survives
      auto set_threshold = [&](unsigned long long tb) {
        thr_bits = tb;
        const double cth = V - __longlong_as_double((long long)tb) - 1e-5;
        s_r = (cth > 0.0) ? __double2float_rd(sqrt(cth) * (1.0 - 1e-9) - eps) : -1.0f;
        if (debug & 128) s_r = INFINITY;  // timing: the max computed, no chunk ever hits (results invalid)
      };
      auto push = [&](uint32_t rel) {
        while (qt - *myhead >= (uint32_t)QCAP) __nanosleep(32);
        myq[qt & (QCAP - 1)] = rel;
        ++qt;
        __threadfence_block();
        *mytail = qt;
      };
      for (int j = (int)((group - (int)(gt % NGRP) + NGRP) % NGRP); j < nt; j += NGRP) {
        const uint32_t gj = gt + (uint32_t)j;
        const int acc = (int)(gj % NACC), acc_ph = (int)((gj / NACC) & 1);
        { long long t0 = TCLK(); mbar_wait_sleep(tfull0 + 8 * acc, acc_ph); tw3 += TCLK() - t0; }
        const bool dbgw = (debug & 32) && blockIdx.x == 0 && kitem == 1 && j < 64 && lane == 0 && (warp == SCR0 || warp == SCR0 + 4);
        if (dbgw) a.dbg[j * 24 + 4] = TCLK();
        fence_after();
        if (!(debug & 4096)) {  // thresholds published by the rescorers
          const unsigned long long tb = thr_s[rk];
          if (tb < thr_bits) set_threshold(tb);
        }
        // slow path of one chunk (rare): seed the row's threshold if it has
        // none, then push the chunk's survivors to the row's queue
        auto slow_path = [&](const float* v, int32_t rel, int32_t e_lo, int32_t e_hi, bool hit) {
          if (FIC_TC_PROF) {  // statistics (profiling builds only: registers are tight)
            ++hit_rounds;
            hit_lanes += hit ? 1 : 0;
          }
          const long long ts0 = TCLK();
          const int32_t wl = max(e_lo, 0), wh = min(e_hi, CH);
          uint64_t wmask = 0;
          if (hit) wmask = ((wh >= 64) ? ~0ull : ((1ull << wh) - 1ull)) & ~((1ull << wl) - 1ull);
          if (hit && thr_bits == 0x7ff0000000000000ull) {  // another group may have seeded the range meanwhile
            const unsigned long long tb = thr_s[rk];
            if (tb < thr_bits) set_threshold(tb);
          }
          const bool seed = hit && thr_bits == 0x7ff0000000000000ull;
          if (__any_sync(0xffffffffu, seed)) {
            if (FIC_TC_PROF) ++seed_rounds;
            double tnew = INFINITY;
            if (seed) {
              float bv = -1.0f;
#pragma unroll
              for (int q = 0; q < CH; ++q) bv = fmaxf(bv, ((wmask >> q) & 1ull) ? fabsf(v[q]) : -1.0f);
              uint64_t eq = 0;
#pragma unroll
              for (int q = 0; q < CH; ++q) eq |= (fabsf(v[q]) == bv) ? (1ull << q) : 0ull;
              const int e = __ffsll((long long)(eq & wmask)) - 1;
              wmask &= ~(1ull << e);
              const int64_t pe = c0 + rel + e;
              tnew = fmax(exact(pe, pool_id(P, pe), row, sr, srr).err, 0.0);
              ++evals;
              push((uint32_t)(rel + e));  // the rescorer records it
            }
            for (int m = 1; m < n_iso; m <<= 1)
              tnew = fmin(tnew, __shfl_xor_sync(0xffffffffu, tnew, m));
            const unsigned long long tb = (unsigned long long)__double_as_longlong(tnew);
            if (tb < thr_bits) {
              set_threshold(tb);
              if (iso == 0 && rvalid) {
                atomicMin(thr_s + rk, tb);
                atomicMin(a.thr_g + rid, tb);
              }
            }
          }
          uint64_t m = 0;
          if (hit) {
#pragma unroll
            for (int q = 0; q < CH; ++q) m |= (fabsf(v[q]) >= s_r || (debug & 64)) ? (1ull << q) : 0ull;
            m &= wmask;
          }
          if (FIC_TC_SL && a.sl && !pilot) {
            // survivors the row's queue cannot take now go to the survivor
            // list as one (row, chunk, mask) entry: the screener never waits
            // for the rescoring warp on a chunk with many survivors
            const uint32_t n = (uint32_t)__popcll(m);
            const bool to_list = list_all ? n > 0 : n > (uint32_t)QCAP - (qt - *myhead);
            const unsigned lm = __ballot_sync(0xffffffffu, to_list);
            if (lm && !sl_dead) {
              const uint32_t cnt = (uint32_t)__popc(lm), left = sl_end - sl_pos;
              const uint32_t k = (uint32_t)__popc(lm & ((1u << lane) - 1u));
              uint32_t idx = sl_pos + k;
              if (cnt > left) {  // warp-uniform: the rest goes to a fresh chunk
                uint32_t nb = 0;
                if (lane == 0) nb = atomicAdd(a.sl_count, (uint32_t)SLCH);
                nb = __shfl_sync(0xffffffffu, nb, 0);
                if (k >= left) idx = nb + (k - left);
                sl_pos = nb + (cnt - left);
                sl_end = nb + SLCH;
                sl_dead = nb >= a.sl_cap;
              } else {
                sl_pos += cnt;
              }
              if (to_list && idx < a.sl_cap) {
                a.sl[idx] = make_uint4((rid << 3) | (uint32_t)iso, (uint32_t)(c0 + rel), (uint32_t)m,
                                       (uint32_t)(m >> 32));
                m = 0;
              }
            }
          }
          while (m) {
            const int e = __ffsll((long long)m) - 1;
            m &= m - 1;
            push((uint32_t)(rel + e));
          }
          tw4 += TCLK() - ts0;
        };
        // hit list: one entry for the warp's hit rows of this chunk (no
        // per-row masks, no seeding: rows without a threshold take slow_path)
        // a slot for one entry in the warp's chunk (refilled when used up)
        auto hl_reserve = [&]() -> bool {
          if (hl_dead) return false;
          if (hl_pos == hl_end) {  // warp-uniform
            uint32_t nb = 0;
            if (lane == 0) nb = atomicAdd(a.hl_count, HLCH);
            nb = __shfl_sync(0xffffffffu, nb, 0);
            hl_pos = nb;
            hl_end = nb + HLCH;
          }
          if (hl_pos >= a.hl_cap) {
            hl_dead = true;
            return false;
          }
          return true;
        };
        auto hl_write = [&](int32_t rel, unsigned bal) {  // into the reserved slot
          if (lane == 0)
            a.hl[hl_pos] = make_uint4((uint32_t)((int64_t)tile * a.RT), (uint32_t)(32 * (warp & 3) + rbase),
                                      (uint32_t)(c0 + rel), bal);
          ++hl_pos;
        };
        // the warp's rows can go to the hit list (no row still needs a seed)
        auto hl_ok = [&](bool hit) {
          return K == 16 && FIC_TC_SL && a.hl && list_all &&
                 !__any_sync(0xffffffffu, hit && thr_bits == 0x7ff0000000000000ull);
        };
        auto hl_append = [&](int32_t rel, bool hit) -> bool {
          const unsigned bal = __ballot_sync(0xffffffffu, hit);
          if (!hl_reserve()) return false;
          hl_write(rel, bal);
          return true;
        };
        auto on_hit = [&](const float* v, int32_t rel, int32_t e_lo, int32_t e_hi, bool hit) {
          if constexpr (DUMP) {
            if (FIC_TC_PROF) {
              ++hit_rounds;
              hit_lanes += hit ? 1 : 0;
            }
            if (hit) {
              const long long ts0 = TCLK();
              const uint32_t t = atomicAdd(const_cast<uint32_t*>(ring_ticket), 1u);
              while (t - *ring_head >= (uint32_t)NSLOT) __nanosleep(32);
              uint32_t* dst = reinterpret_cast<uint32_t*>(ring + (t % NSLOT) * SLOTB);
              const uint32_t win = (uint32_t)max(e_lo, 0) | ((uint32_t)min(e_hi, CH) << 8);
              if constexpr (SLOTW % 4 == 0) {
                float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
                for (int e = 0; e < CH / 4; ++e) d4[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
                *reinterpret_cast<uint4*>(dst + CH) = make_uint4((uint32_t)row, (uint32_t)rel, win, 0u);
              } else {
#pragma unroll
                for (int e = 0; e < CH; ++e) dst[e] = __float_as_uint(v[e]);
                dst[CH] = (uint32_t)row;
                dst[CH + 1] = (uint32_t)rel;
                dst[CH + 2] = win;
              }
              __threadfence_block();
              ring_flag[t % NSLOT] = t + 1;
              if (FIC_TC_DUMP_WAIT && thr_bits == 0x7ff0000000000000ull) {
                // a row without a threshold would copy every chunk of its
                // window until the rescoring warp has seeded it (it does so
                // from this very slot: the chunk has a column of the row's
                // window); waiting here once costs less than that flood
                volatile unsigned long long* tp = thr_s + rk;
                unsigned long long tb = *tp;
                while (tb == 0x7ff0000000000000ull) {
                  __nanosleep(64);
                  tb = *tp;
                }
                set_threshold(tb);
              }
              tw4 += TCLK() - ts0;
            }
            return;
          }
          // (4x4 ranges only: the 8x8 screeners keep their registers)
#if FIC_TC_LEAN
          // experiment: 4x4 main items append every hit chunk to the hit list
          // (rows without a threshold hit on every chunk), no slow path
          if (K == 16 && a.hl && !pil) {
            hl_append(rel, hit);
            return;
          }
#endif
          if (hl_ok(hit) && hl_append(rel, hit)) return;
          slow_path(v, rel, e_lo, e_hi, hit);
        };
        // |u| max of CH values: four FMNMX3 chains
        auto chunk_max = [&](const float* v) {
          float m0 = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fabsf(v[2]));
          float m1 = fmaxf(fmaxf(fabsf(v[3]), fabsf(v[4])), fabsf(v[5]));
          float m2 = fmaxf(fmaxf(fabsf(v[6]), fabsf(v[7])), fabsf(v[8]));
          float m3 = fmaxf(fmaxf(fabsf(v[9]), fabsf(v[10])), fabsf(v[11]));
#pragma unroll
          for (int e = 12; e < CH - 4; e += 8) {
            m0 = fmaxf(fmaxf(m0, fabsf(v[e])), fabsf(v[e + 1]));
            m1 = fmaxf(fmaxf(m1, fabsf(v[e + 2])), fabsf(v[e + 3]));
            m2 = fmaxf(fmaxf(m2, fabsf(v[e + 4])), fabsf(v[e + 5]));
            m3 = fmaxf(fmaxf(m3, fabsf(v[e + 6])), fabsf(v[e + 7]));
          }
          m0 = fmaxf(fmaxf(m0, fabsf(v[CH - 4])), fabsf(v[CH - 3]));
          m1 = fmaxf(fmaxf(m1, fabsf(v[CH - 2])), fabsf(v[CH - 1]));
          return fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
        };
        auto release = [&]() {
          fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader)
              mbar_arrive(tempty0 + 8 * acc);
            else
              mbar_arrive_cluster(map_to_rank(tempty0 + 8 * acc, 0));
          }
        };
        if (F16ACC && !pil) {
          // f16 accumulators: the whole stage in 64 registers with one load
          // and one wait, released at once; packed 3-input |x| max per
          // 64-column chunk; a hit chunk is unpacked to fp32 for the hit path
          uint32_t pk[BN / 2];
          if (!(debug & 1)) tmem_ld64p(lane_base + acc * BN, pk);
          tmem_wait_ld();
          release();
          if (debug & 1) continue;
          auto chunk_max_h = [&](const uint32_t* r) {
            auto hv = [&](int e) { return __habs2(*reinterpret_cast<const __half2*>(r + e)); };
            __half2 m0 = __hmax2(__hmax2(hv(0), hv(1)), hv(2));
            __half2 m1 = __hmax2(__hmax2(hv(3), hv(4)), hv(5));
            __half2 m2 = __hmax2(__hmax2(hv(6), hv(7)), hv(8));
            __half2 m3 = __hmax2(__hmax2(hv(9), hv(10)), hv(11));
#pragma unroll
            for (int e = 12; e < 28; e += 8) {
              m0 = __hmax2(__hmax2(m0, hv(e)), hv(e + 1));
              m1 = __hmax2(__hmax2(m1, hv(e + 2)), hv(e + 3));
              m2 = __hmax2(__hmax2(m2, hv(e + 4)), hv(e + 5));
              m3 = __hmax2(__hmax2(m3, hv(e + 6)), hv(e + 7));
            }
            m0 = __hmax2(__hmax2(m0, hv(28)), hv(29));
            m1 = __hmax2(__hmax2(m1, hv(30)), hv(31));
            const __half2 mm = __hmax2(__hmax2(m0, m1), __hmax2(m2, m3));
            return fmaxf(__low2float(mm), __high2float(mm));
          };
          float mx[BN / CH];
#pragma unroll
          for (int h = 0; h < BN / CH; ++h) mx[h] = chunk_max_h(pk + (CH / 2) * h);
#pragma unroll
          for (int h = 0; h < BN / CH; ++h) {
            const int32_t rel = j * BN + CH * h;
            const int32_t e_lo = lo32 - rel, e_hi = hi32 - rel;
            const bool in_window = (uint32_t)(e_hi - 1) < (uint32_t)(hi32 - lo32 + CH - 1);
            const bool hit = !(debug & 8) & in_window & !rflat & (mx[h] >= s_r);
            if (__any_sync(0xffffffffu, hit)) {
              // (converting inside the hit path instead of this fp32 copy
              // spilled in the screening loop: 5.65 -> 6.26 ms at cfg3)
              float v[CH];
#pragma unroll
              for (int e = 0; e < CH / 2; ++e) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(pk + (CH / 2) * h + e));
                v[2 * e] = f.x;
                v[2 * e + 1] = f.y;
              }
              on_hit(v, rel, e_lo, e_hi, hit);
            }
          }
        } else if constexpr (WIDE) {
          // the whole stage in registers: loads, release, independent chunk maxima
          float v[SW];
          if (!(debug & 1)) {
#pragma unroll
            for (int c = 0; c < SW / 32; ++c) tmem_ld32(lane_base + acc * BN + slice * SW + 32 * c, v + 32 * c);
          }
          tmem_wait_ld();
          release();
          if (debug & 1) continue;
          float mx[SW / CH];
#pragma unroll
          for (int h = 0; h < SW / CH; ++h) mx[h] = chunk_max(v + CH * h);
#pragma unroll
          for (int h = 0; h < SW / CH; ++h) {
            const int32_t rel = j * BN + slice * SW + CH * h;
            const int32_t e_lo = lo32 - rel, e_hi = hi32 - rel;
            const bool hit = !(debug & 8) & rvalid & !rflat & (e_lo < CH) & (e_hi > 0) & (mx[h] >= s_r);
            if (__any_sync(0xffffffffu, hit)) on_hit(v + CH * h, rel, e_lo, e_hi, hit);
          }
        } else {
#pragma unroll
          for (int h = 0; h < SW / CH; ++h) {
            float v[CH];
            if (!(debug & 1)) {
#pragma unroll
              for (int c = 0; c < CH / 32; ++c)
                tmem_ld32(lane_base + acc * BN + slice * SW + CH * h + 32 * c, v + 32 * c);
            }
            tmem_wait_ld();
            if (dbgw) a.dbg[j * 24 + 5 + h] = TCLK();
            if (h == SW / CH - 1) release();  // release the stage before screening its last chunk
            if (debug & 1) continue;
            const int32_t rel = j * BN + slice * SW + CH * h;  // chunk start, relative to c0
            const int32_t e_lo = lo32 - rel, e_hi = hi32 - rel;
            const float mx = chunk_max(v);
            // bitwise, so the max is computed unconditionally (no branch around it)
            // [rel, rel + CH) meets [lo32, hi32) (hi32 > lo32 when valid): one unsigned compare
            const bool in_window = (uint32_t)(e_hi - 1) < (uint32_t)(hi32 - lo32 + CH - 1);
            const bool hit = !(debug & 8) & in_window & !rflat & (mx >= s_r);
            if (__any_sync(0xffffffffu, hit)) on_hit(v, rel, e_lo, e_hi, hit);
          }
        }
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicAdd((uint32_t*)edone, 1u);
    } else if (is_res) {
      // ------------------------------ rescoring ------------------------------
      // Thread t owns rows t + RSTRIDE * h: it drains their survivor queues,
      // evaluates each candidate exactly (state in shared memory) and
      // publishes the range's threshold.
      const int t = (int)threadIdx.x - 32 * RES0;
#pragma unroll
      for (int h = 0; h < RROWS; ++h) {
        const int r = t + RSTRIDE * h, k = (r + rbase) / n_iso;
        const int64_t g = (int64_t)tile * a.RT + k;
        RowState st;
        st.err = INFINITY;
        st.pre = INFINITY;
        st.dom = 0xffffffffu;
        st.sq = st.oq = 0;
        st.iso = (uint8_t)(r + rbase - k * n_iso);
        st.valid = (k < a.RT && g < n_tr) ? 1 : 0;
        st.sr = st.srr = 0.0;
        if (st.valid) {
          const RangeInfo inf = Rv.info[tlist[g]];
          st.sr = inf.sr;
          st.srr = inf.srr;
        }
        rstate[r] = st;
      }
      uint32_t hd[RROWS * NSLICE];
#pragma unroll
      for (int q = 0; q < RROWS * NSLICE; ++q) hd[q] = 0;
      // two candidates per pass (from any of the thread's queues), evaluated
      // back to back so their fp64 chains overlap; updates applied in order
      auto apply = [&](int r, const Cand& cd, uint32_t did) {
        const int k = r / n_iso;
        RowState st = rstate[r];
        st.pre = fmin(st.pre, cd.pre);
        if (better(cd.err, did, st.iso, st.err, st.dom, st.iso)) {
          st.err = cd.err;
          st.dom = did;
          st.sq = (uint8_t)cd.sq;
          st.oq = (uint8_t)cd.oq;
        }
        rstate[r] = st;
        const unsigned long long eb = (unsigned long long)__double_as_longlong(fmax(cd.err, 0.0));
        if (eb < thr_s[k]) {  // an improvement: publish to the screeners and the other segments
          atomicMin(thr_s + k, eb);
          atomicMin(a.thr_g + s_rid[k], eb);
        }
      };
      constexpr int NE = 4;  // candidates per lane and pass
      if constexpr (DUMP) {
        // hit ring consumer: up to 32 slots per pass, in ticket order (the
        // ready prefix of the next 32 tickets), the warp's lanes split evenly
        // over the pass's slots: they filter the chunk's 64 values against
        // the row's freshest threshold (a row without one first evaluates
        // the chunk's best |u|), the slots are handed back, the survivors
        // are evaluated exactly and the lanes' results merged per row
        // (lowest lane of each row)
        constexpr unsigned long long INF_BITS = 0x7ff0000000000000ull;
        uint32_t next = 0;
        while (true) {
          const uint32_t myt = next + (uint32_t)t, sl = myt % NSLOT;
          const unsigned rb = __ballot_sync(0xffffffffu, ring_flag[sl] == myt + 1);
          const int n = rb == 0xffffffffu ? 32 : __ffs((int)~rb) - 1;
          if (n == 0) {
            if (*edone == (uint32_t)NEPI) {
              __threadfence_block();
              if (*ring_ticket == next) break;  // every ticket taken has been consumed
            } else {
              __nanosleep(FIC_TC_RES_SLEEP);
            }
            continue;
          }
          __threadfence_block();  // the slots' data behind their flags
          // L lanes per slot (a power of two, 32 for one slot .. 1 for 17-32
          // slots), each CH / L columns... the usual pass has one or two slots,
          // and a single lane sweeping 64 values would cost the warp (and the
          // screening warps sharing its scheduler) 64 iterations of issue slots
          int lg = 0;  // log2(slots rounded up to a power of two)
          while ((1 << lg) < n) ++lg;
          const int L = 32 >> lg, cpl = CH / L;  // lanes per slot, columns per lane (2 .. 64)
          const int si = t >> (5 - lg), sub = t & (L - 1);
          const bool act = si < n;
          const uint32_t* sw = reinterpret_cast<const uint32_t*>(ring + ((next + (uint32_t)si) % NSLOT) * SLOTB);
          int r = 0, wl = 0, wh = 0;
          int32_t rel = 0;
          if (act) {
            r = (int)sw[CH];
            rel = (int32_t)sw[CH + 1];
            wl = (int)(sw[CH + 2] & 255u);
            wh = (int)(sw[CH + 2] >> 8);
          }
          const int k = r / n_iso;
          const double e_sr = rstate[r].sr, e_srr = rstate[r].srr, Vr = rowV[r], er = rowEps[r];
          unsigned long long tb = thr_s[k];
          double b_err = INFINITY, b_pre = INFINITY;
          uint32_t b_dom = 0xffffffffu, b_q = 0;
          auto take = [&](int c) {  // exact evaluation of column c of the chunk into the lane's best
            const int64_t p = c0 + rel + c;
            const uint32_t id = pool_id(P, p);
            const Cand cd = exact(p, id, r, e_sr, e_srr);
            b_pre = fmin(b_pre, cd.pre);
            if (better(cd.err, id, 0, b_err, b_dom, 0)) {
              b_err = cd.err;
              b_dom = id;
              b_q = (uint32_t)cd.sq | ((uint32_t)cd.oq << 8);
            }
            ++evals;
          };
          auto s_of = [&](unsigned long long bits) -> float {
            const double cth = Vr - __longlong_as_double((long long)bits) - 1e-5;
            return (bits != INF_BITS && cth > 0.0) ? __double2float_rd(sqrt(cth) * (1.0 - 1e-9) - er) : -1.0f;
          };
          float s_r = s_of(tb);
          const int q0 = sub * cpl;
          uint64_t mask = 0;  // bit q - q0: column q survives
          float bestv = -1.0f;
          int bestc = -1;
          if (act) {
            for (int q = q0; q < q0 + cpl; ++q) {
              const float v = fabsf(__uint_as_float(sw[q]));
              const bool inw = q >= wl && q < wh;
              if (inw && v > bestv) {
                bestv = v;
                bestc = q;
              }
              mask |= (inw && v >= s_r) ? (1ull << (q - q0)) : 0ull;
            }
          }
          if (__any_sync(0xffffffffu, act && tb == INF_BITS)) {
            // a range without a threshold: the chunk's best |u| (over the
            // slot's L lanes) is evaluated first, the rest filtered against it
            float gv = bestv;
            for (int m = 1; m < L; m <<= 1) gv = fmaxf(gv, __shfl_xor_sync(0xffffffffu, gv, m));
            const bool noth = act && tb == INF_BITS && gv >= 0.0f;
            // the slot's lowest lane holding the maximum evaluates it
            const unsigned cand = __ballot_sync(0xffffffffu, noth && bestv == gv);
            const unsigned mine = cand & (L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (t & ~(L - 1))));
            const int first = __ffs((int)mine) - 1;
            double e0 = INFINITY;
            if (noth && t == first) {
              take(bestc);
              e0 = b_err;
            }
            e0 = __shfl_sync(0xffffffffu, e0, first < 0 ? 0 : first);
            if (noth) {
              tb = (unsigned long long)__double_as_longlong(fmax(e0, 0.0));
              s_r = s_of(tb);
              mask = 0;
              for (int q = q0; q < q0 + cpl; ++q) {
                const float v = fabsf(__uint_as_float(sw[q]));
                mask |= (q >= wl && q < wh && !(t == first && q == bestc) && v >= s_r) ? (1ull << (q - q0)) : 0ull;
              }
            }
          }
          __syncwarp();
          next += (uint32_t)n;
          if (t == 0) *ring_head = next;  // the slots of this pass are free again
          while (mask) {
            const int c = __ffsll((long long)mask) - 1;
            mask &= mask - 1;
            take(q0 + c);
          }
          // merge per row: the lowest lane of each row applies its lanes' results
          const bool has = act && b_dom != 0xffffffffu;
          const unsigned hb = __ballot_sync(0xffffffffu, has);
          if (!hb) continue;
          if (FIC_TC_RES_DIRECT && (hb & (hb - 1)) == 0) {  // one lane holds the pass's only results
            if (has) {
              RowState st = rstate[r];
              st.pre = fmin(st.pre, b_pre);
              if (better(b_err, b_dom, st.iso, st.err, st.dom, st.iso)) {
                st.err = b_err;
                st.dom = b_dom;
                st.sq = (uint8_t)(b_q & 255u);
                st.oq = (uint8_t)(b_q >> 8);
              }
              rstate[r] = st;
              const unsigned long long eb = (unsigned long long)__double_as_longlong(fmax(st.err, 0.0));
              if (eb < thr_s[k]) {
                atomicMin(thr_s + k, eb);
                atomicMin(a.thr_g + s_rid[k], eb);
              }
            }
            __syncwarp();
            continue;
          }
          s_cerr[t] = b_err;
          s_cpre[t] = b_pre;
          s_cdom[t] = b_dom;
          s_csqoq[t] = b_q;
          __syncwarp();
          const unsigned grp = __match_any_sync(0xffffffffu, has ? (uint32_t)r : (0x80000000u | (uint32_t)t));
          if (has && t == __ffs((int)grp) - 1) {
            RowState st = rstate[r];
            unsigned g2 = grp;
            while (g2) {
              const int j = __ffs((int)g2) - 1;
              g2 &= g2 - 1;
              st.pre = fmin(st.pre, s_cpre[j]);
              if (better(s_cerr[j], s_cdom[j], st.iso, st.err, st.dom, st.iso)) {
                st.err = s_cerr[j];
                st.dom = s_cdom[j];
                st.sq = (uint8_t)(s_csqoq[j] & 255u);
                st.oq = (uint8_t)(s_csqoq[j] >> 8);
              }
            }
            rstate[r] = st;
            const unsigned long long eb = (unsigned long long)__double_as_longlong(fmax(st.err, 0.0));
            if (eb < thr_s[k]) {  // an improvement: publish to the screeners and the other segments
              atomicMin(thr_s + k, eb);
              atomicMin(a.thr_g + s_rid[k], eb);
            }
          }
          __syncwarp();
        }
      } else {
#if FIC_TC_BAL
      // Balanced drain: the warp is the single consumer of all 2 x 128
      // queues; each pass takes up to 32 x NE pending entries from any rows
      // (lane-major prefix sum over the lanes' queues), so every lane
      // evaluates even when the survivors sit in a few rows.  Heads advance
      // only after every lane has read its entries (each head keeps one
      // writer: its owner lane); results of the same row are merged by the
      // row's lowest lane in that pass (one writer per row state).
      constexpr int Q = RROWS * NSLICE;
      static_assert(NRES == 1, "the balanced drain is one warp");
      while (true) {
        uint32_t pend[Q], mine = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int r = t + RSTRIDE * (q / NSLICE), qs = q % NSLICE;
          pend[q] = qtail[r * NSLICE + qs] - hd[q];
          mine += pend[q];
        }
        uint32_t incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
          if (t >= d) incl += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) {
          if (*edone == (uint32_t)NEPI) {
            __threadfence_block();
            bool empty = true;
#pragma unroll
            for (int q = 0; q < Q; ++q)
              empty = empty && (hd[q] == qtail[(t + RSTRIDE * (q / NSLICE)) * NSLICE + q % NSLICE]);
            if (__all_sync(0xffffffffu, empty)) break;
          } else {
            __nanosleep(256);
          }
          continue;
        }
        __threadfence_block();  // the entries behind the tails we read
        s_incl[t] = incl;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          s_pend[t * Q + q] = pend[q];
          s_hd[t * Q + q] = hd[q];
        }
        __syncwarp();
        const uint32_t take = min(total, (uint32_t)(32 * NE));
        Cand cd[NE];
        uint32_t did[NE];
        int rr[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const uint32_t tt = min((uint32_t)t + 32u * e, take - 1);  // (duplicates are not applied)
          int o = 0;  // owner lane: the first whose inclusive count exceeds tt
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1)
            if (s_incl[o + step - 1] <= tt) o += step;
          uint32_t k = tt - (o ? s_incl[o - 1] : 0u);
          int q = 0;
          while (k >= s_pend[o * Q + q]) {
            k -= s_pend[o * Q + q];
            ++q;
          }
          const int r = o + RSTRIDE * (q / NSLICE), qs = q % NSLICE;
          const uint32_t rel = qbuf[(r * NSLICE + qs) * QCAP + ((s_hd[o * Q + q] + k) & (QCAP - 1))];
          const int64_t p = c0 + rel;
          rr[e] = r;
          did[e] = pool_id(P, p);
          cd[e] = exact(p, did[e], r, rstate[r].sr, rstate[r].srr);
        }
        __syncwarp();  // every entry of this pass has been read
        {
          const uint32_t excl = incl - mine;
          uint32_t cons = take > excl ? min(mine, take - excl) : 0u;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const uint32_t c = min(pend[q], cons);
            cons -= c;
            if (c) {
              hd[q] += c;
              qhead[(t + RSTRIDE * (q / NSLICE)) * NSLICE + q % NSLICE] = hd[q];
            }
          }
        }
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const bool ok = (uint32_t)t + 32u * e < take;
          s_crow[t] = ok ? (uint32_t)rr[e] : 0xffffffffu;
          s_cerr[t] = cd[e].err;
          s_cpre[t] = cd[e].pre;
          s_cdom[t] = did[e];
          s_csqoq[t] = (uint32_t)cd[e].sq | ((uint32_t)cd[e].oq << 8);
          __syncwarp();
          const unsigned grp = __match_any_sync(0xffffffffu, s_crow[t]);
          if (ok && t == __ffs(grp) - 1) {  // the row's lowest lane merges its pass results
            const int r = rr[e];
            RowState st = rstate[r];
            unsigned g2 = grp;
            while (g2) {
              const int j = __ffs(g2) - 1;
              g2 &= g2 - 1;
              const double ej = s_cerr[j];
              const uint32_t dj = s_cdom[j];
              st.pre = fmin(st.pre, s_cpre[j]);
              if (better(ej, dj, st.iso, st.err, st.dom, st.iso)) {
                st.err = ej;
                st.dom = dj;
                st.sq = (uint8_t)(s_csqoq[j] & 255u);
                st.oq = (uint8_t)(s_csqoq[j] >> 8);
              }
            }
            rstate[r] = st;
            const int k = r / n_iso;
            const unsigned long long eb = (unsigned long long)__double_as_longlong(fmax(st.err, 0.0));
            if (eb < thr_s[k]) {  // an improvement: publish to the screeners and the other segments
              atomicMin(thr_s + k, eb);
              atomicMin(a.thr_g + s_rid[k], eb);
            }
          }
          __syncwarp();
        }
        evals += (uint32_t)t < take ? min((take - 1 - (uint32_t)t) / 32u + 1u, (uint32_t)NE) : 0u;
      }
#else
      while (true) {
        int got[NE];
        uint32_t rel[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          got[e] = -1;
          rel[e] = 0;
        }
        int ng = 0;
#pragma unroll
        for (int q = 0; q < RROWS * NSLICE; ++q) {
          const int r = t + RSTRIDE * (q / NSLICE), qs = q % NSLICE;
          const uint32_t tl = qtail[r * NSLICE + qs];
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            if (ng == e && hd[q] != tl) {
              __threadfence_block();
              rel[e] = qbuf[(r * NSLICE + qs) * QCAP + (hd[q] & (QCAP - 1))];
              qhead[r * NSLICE + qs] = ++hd[q];
              got[e] = q / NSLICE;
              ++ng;
            }
          }
        }
        if (ng > 0) {
          Cand cd[NE];
          uint32_t did[NE];
          int rr[NE];
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            rr[e] = got[e] >= 0 ? t + RSTRIDE * got[e] : t + RSTRIDE * got[0];
            const int64_t p = c0 + (got[e] >= 0 ? rel[e] : rel[0]);
            did[e] = pool_id(P, p);
            cd[e] = exact(p, did[e], rr[e], rstate[rr[e]].sr, rstate[rr[e]].srr);
          }
#pragma unroll
          for (int e = 0; e < NE; ++e)
            if (e < ng) apply(rr[e], cd[e], did[e]);
          evals += ng;
        } else if (*edone == (uint32_t)NEPI) {
          __threadfence_block();
          bool empty = true;
#pragma unroll
          for (int q = 0; q < RROWS * NSLICE; ++q)
            empty = empty && (hd[q] == qtail[(t + RSTRIDE * (q / NSLICE)) * NSLICE + q % NSLICE]);
          if (empty) break;
        } else {
          __nanosleep(256);
        }
      }
#endif
      }
      __syncwarp();
      // combine the n_iso rows of each range: lexicographic (err, dom, iso)
#pragma unroll
      for (int h = 0; h < RROWS; ++h) {
        const int r = t + RSTRIDE * h;
        const RowState st = rstate[r];
        double err = st.err, pre = st.pre;
        uint32_t dom = st.dom;
        int biso = st.iso, sq = st.sq, oq = st.oq;
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
        if (st.iso == 0 && st.valid && !pil) {
          const int64_t g = (int64_t)tile * a.RT + (r + rbase) / n_iso;
          Partial out;
          out.err = err;
          out.pre = pre;
          out.dom = dom;
          out.iso = (uint8_t)biso;
          out.sq = (uint8_t)sq;
          out.oq = (uint8_t)oq;
          out.valid = (dom != 0xffffffffu) ? 1 : 0;
          Partial* dst = a.partials + a.slot_base[tlist[g]] + slot;
          *dst = out;
          if (it - n_pilot < n_whole)  // a whole segment: its piece slots stay empty
            for (int q = 1; q < a.nsub; ++q) dst[q].valid = 0;
        }
      }
    }
    gt += (uint32_t)nt;
    ++kitem;
    const long long ti2 = TCLK();
    cta_sync<CG>();
    if (warp == 0) tteardown += TCLK() - ti2;
    (void)ti1;
  }

  if (FIC_TC_SL && is_scr && a.sl) {  // unused tail of the warp's chunk: empty entries
    for (uint32_t i = sl_pos + lane; i < min(sl_end, a.sl_cap); i += 32) a.sl[i] = make_uint4(0, 0, 0, 0);
  }
  if (K == 16 && FIC_TC_SL && is_scr && a.hl) {
    for (uint32_t i = hl_pos + lane; i < min(hl_end, a.hl_cap); i += 32) a.hl[i] = make_uint4(0, 0, 0, 0);
  }
  if (is_res || is_scr) {
    for (int m = 16; m >= 1; m >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, m);
    if (lane == 0) atomicAdd(a.counters, evals);
    if (lane == 0 && seed_rounds) atomicAdd(a.counters + 14, seed_rounds);  // warp-level seeding rounds
    if (!DBG && FIC_TC_PROF) {  // hit statistics (warp-level rounds, lanes)
      for (int m = 16; m >= 1; m >>= 1) hit_lanes += __shfl_xor_sync(0xffffffffu, hit_lanes, m);
      if (lane == 0 && hit_rounds) {
        atomicAdd(a.counters + 12, hit_rounds);
        atomicAdd(a.counters + 13, hit_lanes);
      }
    }
    if (((debug & 4) || FIC_TC_PROF) && lane == 0 && is_scr) {
      atomicAdd(a.counters + 7, (unsigned long long)tw3);
      atomicAdd(a.counters + 8, (unsigned long long)tw4);
      atomicAdd(a.counters + 9, (unsigned long long)(TCLK() - tstart));
    }
  }
  if (((debug & 4) || FIC_TC_PROF) && lane == 0 && warp == 0) {
    atomicAdd(a.counters + 4, (unsigned long long)tw0);
    atomicAdd(a.counters + 11, (unsigned long long)tsetup);
    atomicAdd(a.counters + 12, (unsigned long long)tteardown);
    atomicAdd(a.counters + 13, (unsigned long long)nitems);
  }
  if (((debug & 4) || FIC_TC_PROF) && lane == 0 && warp == 1) {
    atomicAdd(a.counters + 10, (unsigned long long)(TCLK() - tstart));
    atomicAdd(a.counters + 5, (unsigned long long)tw1);
    atomicAdd(a.counters + 6, (unsigned long long)tw2);
  }
  cta_sync<CG>();
  if (DBG && (debug & 8192) && threadIdx.x == 0) {
    unsigned long long gt_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_end));
    a.dbg[2 * blockIdx.x] = gt_start;
    a.dbg[2 * blockIdx.x + 1] = gt_end;
    a.dbg[1024 + blockIdx.x] = (unsigned long long)nitems;
  }
  if (warp == 0) {
    fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
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

// rows per tensor tile (the planner sizes tiles with it)
static int tc_cg(int K) {
  if (K != 64) return 1;
  const char* e = getenv("FIC_TC_CG");
  return (e && atoi(e) == 2) ? 2 : 1;
}
int tc_tile_rows(int K) { return BM * tc_cg(K); }

template <int K, int CG, int SRC>
static void launch_tc_k(const PoolView& P, const RangeView& Rv, const TcArgs& a, cudaStream_t s) {
  using C = Cfg<K, CG>;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)P.D};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)K, (cuuint32_t)(BN / CG)};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)P.bh, dims, strides,
                             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             K == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) throw Error{FIC_ECUDA, "cuTensorMapEncodeTiled failed"};
  smem_optin_k(k_match_tc<K, CG, false, SRC>, C::SMEM);
  smem_optin_k(k_match_tc<K, CG, true, SRC>, C::SMEM);
  int dev = 0, sms = 148;
  FIC_CUDA(cudaGetDevice(&dev));
  FIC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t clusters = std::min<int64_t>(a.n_items + a.n_split * (a.nsub - 1), sms / CG);
  TcArgs aa = a;
  const char* dbg = getenv("FIC_TC_DEBUG");
  aa.debug = dbg ? atoi(dbg) : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * CG));
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (aa.debug)
    FIC_CUDA(cudaLaunchKernelEx(&cfg, k_match_tc<K, CG, true, SRC>, map, P, Rv, aa));
  else
    FIC_CUDA(cudaLaunchKernelEx(&cfg, k_match_tc<K, CG, false, SRC>, map, P, Rv, aa));
  FIC_CHECK_LAUNCH();
}

void launch_tc(const PoolView& P, const RangeView& Rv, const TcArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  // one instantiation per domain source (DomSrc): row segments or box planes
  const bool trows = P.src.trows != nullptr;
  if (!trows && !P.src.planes) invalid("tensor matcher needs the row segments or box planes");
  if (Rv.K == 64 && tc_cg(64) == 2) {
    if (trows)
      launch_tc_k<64, 2, SRC_TROWS>(P, Rv, a, s);
    else
      launch_tc_k<64, 2, SRC_PLANES>(P, Rv, a, s);
  } else if (Rv.K == 64) {
    if (trows)
      launch_tc_k<64, 1, SRC_TROWS>(P, Rv, a, s);
    else
      launch_tc_k<64, 1, SRC_PLANES>(P, Rv, a, s);
  } else if (Rv.K == 16) {
    launch_tc_k<16, 1, SRC_PLANES>(P, Rv, a, s);
  } else {
    invalid("tensor matcher supports range_size 4 and 8");
  }
}

}  // namespace fic
