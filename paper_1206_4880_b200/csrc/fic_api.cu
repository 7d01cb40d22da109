// C ABI of the B200 fractal encoder (include/fic_b200.h): validation, pool
// planning, work decomposition and orchestration of the kernels.
#include <cuda.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "kernels.h"
#include "match.h"

extern char** environ;  // the process environment (graphs_allowed)

namespace fic {

static thread_local std::string g_err;
thread_local int g_launches = 0;
void set_error(const std::string& m) { g_err = m; }
const char* last_error() { return g_err.c_str(); }

// The attribute is per (device, function) and only ever raised: a launch
// with less dynamic shared memory than the current limit is always valid,
// while lowering it would break a later, larger launch of the same kernel.
void smem_optin(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> limit;
  int dev = 0;
  FIC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int& cur = limit[{dev, func}];
  if (bytes <= cur) return;
  FIC_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cur = bytes;
}

// ---------------------------------------------------------------------------
// stream-ordered scratch: a call's buffers are bump-allocated from an arena
// kept per (thread, device, stream) across calls, so a repeated encode makes
// no allocation at all.  The arena grows (stream-ordered free + malloc from
// the device's default pool) when a call needed more; reuse by the next call
// on the same stream is ordered after this call's kernels by the stream.
// ---------------------------------------------------------------------------
struct Arena {
  char* base = nullptr;
  size_t cap = 0, want = 0;
  bool busy = false;
};
static thread_local std::map<std::pair<int, cudaStream_t>, Arena> g_arenas;

class Scratch {
 public:
  explicit Scratch(cudaStream_t s) : s_(s), guard_(getenv("FIC_ARENA_GUARD") != nullptr) {
    // keep freed blocks cached in the device's default pool (once per device)
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    FIC_CUDA(cudaGetDevice(&dev));
    {
      std::lock_guard<std::mutex> lock(mu);
      if (!done.count(dev)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          uint64_t thr = UINT64_MAX;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        done.insert(dev);
      }
    }
    Arena& ar = g_arenas[{dev, s}];
    if (!ar.busy && !getenv("FIC_NO_ARENA")) {
      ar.busy = true;
      if (ar.cap < ar.want) {  // grow: the last call on this stream needed more
        if (ar.base) FIC_CUDA(cudaFreeAsync(ar.base, s_));
        ar.base = nullptr;
        ar.cap = 0;
        const size_t cap = ar.want + ar.want / 4;
        FIC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ar.base), cap, s_));
        ar.cap = cap;
      }
      arena_ = &ar;
    }
  }
  ~Scratch() {
    for (void* p : ptrs_) cudaFreeAsync(p, s_);
    if (arena_) {
      arena_->want = std::max(arena_->want, used_);
      arena_->busy = false;
    }
  }
  // graph capture support: the bump offset (restored on replay), whether the
  // arena already fits a call the size of the previous ones, whether any
  // allocation fell outside it
  size_t offset() const { return off_; }
  void restore(size_t o) {
    off_ = o;
    used_ = std::max(used_, o);
  }
  bool fits() const { return arena_ && arena_->want > 0 && arena_->cap >= arena_->want; }
  bool spilled() const { return !ptrs_.empty(); }
  const void* arena_base() const { return arena_ ? arena_->base : nullptr; }
  size_t arena_cap() const { return arena_ ? arena_->cap : 0; }
  template <class T>
  T* get(size_t n) {
    if (n == 0) n = 1;
    // FIC_ARENA_GUARD (a home-made write check; compute-sanitizer is not
    // available on every box): each buffer is followed by a red zone -- its
    // alignment slack plus GUARD bytes -- filled with a pattern that verify()
    // expects to find intact after the call's kernels
    const size_t bytes = align_up(n * sizeof(T), 256) + (guard_ ? GUARD : 0);
    used_ += bytes;
    char* p = nullptr;
    if (arena_ && off_ + bytes <= arena_->cap) {
      p = arena_->base + off_;
      off_ += bytes;
    } else {  // beyond the arena: a pool allocation freed at the end
      FIC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, s_));
      ptrs_.push_back(p);
    }
    if (guard_) {
      const size_t live = align_up(n * sizeof(T), 16);  // vector stores may round a tail up to 16 B
      FIC_CUDA(cudaMemsetAsync(p + live, 0xA5, bytes - live, s_));
      zones_.push_back({p + live, bytes - live, n * sizeof(T)});
    }
    return reinterpret_cast<T*>(p);
  }
  // FIC_ARENA_GUARD: every red zone still holds its pattern (call with the
  // call's streams synchronised); throws naming the buffer otherwise
  void verify(const char* what) {
    if (!guard_) return;
    std::vector<unsigned char> h;
    for (size_t i = 0; i < zones_.size(); ++i) {
      const Zone& z = zones_[i];
      h.resize(z.len);
      FIC_CUDA(cudaMemcpy(h.data(), z.at, z.len, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < z.len; ++k)
        if (h[k] != 0xA5) {
          char msg[200];
          snprintf(msg, sizeof(msg),
                   "FIC_ARENA_GUARD: %s wrote past scratch buffer #%zu (%zu bytes): red-zone byte +%zu = 0x%02x",
                   what, i, z.size, k, (unsigned)h[k]);
          throw std::runtime_error(msg);
        }
    }
    guard_checked_ += zones_.size();
  }
  size_t guard_checked() const { return guard_checked_; }

 private:
  static constexpr size_t GUARD = 256;
  struct Zone {
    const char* at;
    size_t len, size;
  };
  cudaStream_t s_;
  Arena* arena_ = nullptr;
  size_t off_ = 0, used_ = 0;
  std::vector<void*> ptrs_;
  bool guard_ = false;
  std::vector<Zone> zones_;
  size_t guard_checked_ = 0;
};

struct Timer {
  cudaEvent_t* ev;
  int n = 0;
  cudaStream_t& s;  // the stream the call currently enqueues on (a graph capture switches it)
  // events are created once per thread and device and reused
  explicit Timer(cudaStream_t& st) : s(st) {
    static thread_local std::map<int, std::vector<cudaEvent_t>> pool;
    int dev = 0;
    FIC_CUDA(cudaGetDevice(&dev));
    auto& v = pool[dev];
    if (v.empty()) {
      v.resize(24);
      for (auto& e : v) FIC_CUDA(cudaEventCreate(&e));
    }
    ev = v.data();
  }
  // external: inside a CUDA graph capture the record becomes a timestamp
  // node (outside a capture it is an ordinary record)
  void mark() { FIC_CUDA(record_timing_event(ev[n++], s)); }
  double ms(int a, int b) {
    float t = 0;
    cudaEventElapsedTime(&t, ev[a], ev[b]);
    return t;
  }
};

// Side stream (one per thread and device): the pool builder and the range
// preparation run on it, overlapping the FD sort and the work planning on
// the caller's stream; event-ordered both ways.
struct SideStream {
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev[6] = {};  // 0 fork (after ranges alloc), 1 fork (order ready), 2 join, 3..5 pool timing
  static SideStream& get() {
    static thread_local std::map<int, SideStream> m;
    int dev = 0;
    FIC_CUDA(cudaGetDevice(&dev));
    SideStream& ss = m[dev];
    if (!ss.s2) {
      FIC_CUDA(cudaStreamCreateWithFlags(&ss.s2, cudaStreamNonBlocking));
      for (auto& e : ss.ev) FIC_CUDA(cudaEventCreate(&e));
    }
    return ss;
  }
};

static const char* kStrategyTuple = "('exhaustive', 'nosearch', 'static2', 'dynamic_fd')";

// Validation in the reference's order (codec.py:313-331, blocks.py:63-68,
// 148-151, fdim.py:48-56) with its messages.
static Geo validate(int H, int W, const fic_params_t& p) {
  if (H <= 0 || W <= 0) invalid("image must be a 2-D uint8 array");
  if (p.strategy < 0 || p.strategy > 3)
    invalid("unknown strategy " + std::to_string(p.strategy) + "; use one of " + kStrategyTuple);
  if (p.domain_size != 2 * p.range_size) invalid("domain_size must be exactly twice range_size");
  if (p.fd_source != 0 && p.fd_source != 1)
    invalid("fd_source must be 'original' or 'downsampled'");
  if (p.range_size <= 0 || H % p.range_size || W % p.range_size)
    invalid("image " + std::to_string(W) + "x" + std::to_string(H) +
            " not divisible by range size " + std::to_string(p.range_size));
  if (p.stride < 1) invalid("stride must be >= 1");
  if (p.domain_size > std::min(W, H))
    invalid("domain size " + std::to_string(p.domain_size) + " exceeds image " +
            std::to_string(W) + "x" + std::to_string(H));
  Geo g;
  g.H = H;
  g.W = W;
  g.rs = p.range_size;
  g.ds = p.domain_size;
  g.st = p.stride;
  g.npx = g.rs * g.rs;
  g.nrx = W / g.rs;
  g.nry = H / g.rs;
  g.R = g.nrx * g.nry;
  g.ndx = (W - g.ds) / g.st + 1;
  g.ndy = (H - g.ds) / g.st + 1;
  g.D = (int64_t)g.ndx * g.ndy;
  g.n_iso = p.isometries ? 8 : 1;
  if (g.D == 0) invalid("empty domain set");
  if (g.D >= (int64_t)1 << 31) invalid("too many domain positions for this build (>= 2^31)");
  return g;
}

// fdim.py:48-56: the DBC estimator needs at least two scales (scale_set)
static void check_dbc_side(int side) {
  int J = 0;
  for (int s = 2; s <= side / 2; s *= 2)
    if (side % s == 0) ++J;
  if (J < 2)
    invalid("block side " + std::to_string(side) + " too small: need at least two DBC scales");
}

// Device-resident DBC tables for one block side.
struct DbcTables {
  int J = 0, smax = 0, ln_len = 0;
  uint16_t* quot = nullptr;
  double* ln = nullptr;
  double* w = nullptr;
  double hw[7] = {};   // host copies: slope weights, max count increment per scale
  int hqmax[7] = {};
  int qshift[7] = {-1, -1, -1, -1, -1, -1, -1};  // quotient table == v >> qshift (else -1)
  const std::vector<double>* hln = nullptr;  // host copy of the ln table (cached, never freed)
};

static DbcTables make_dbc(Scratch& sc, cudaStream_t s, int side, const double* h_ln, int ln_len,
                          const double* h_w, int n_w, int gray_levels = 256) {
  DbcTables t;
  std::vector<uint16_t> q(7 * 256);
  int need = 0;
  t.J = dbc_tables(side, q.data(), &t.smax, &need, gray_levels);
  if (t.J < 2)
    invalid("block side " + std::to_string(side) + " too small: need at least two DBC scales");
  // ln table: caller's numpy values if long enough, else C log()
  std::vector<double> ln;
  if (h_ln && ln_len >= need) {
    ln.assign(h_ln, h_ln + need);
  } else {
    ln.resize(need);
    for (int k = 0; k < need; ++k) ln[k] = std::log((double)k);
  }
  // slope weights: caller's numpy values, else fdim.py:37-41 in C
  std::vector<double> w(t.J);
  if (h_w && n_w == t.J) {
    std::copy(h_w, h_w + t.J, w.begin());
  } else {
    std::vector<double> xs(t.J);
    double mean = 0;
    for (int j = 0; j < t.J; ++j) {
      xs[j] = std::log((double)side / (double)(2 << j));
      mean = (j == 0) ? xs[0] : mean + xs[j];
    }
    mean /= t.J;
    double dd = 0;
    for (int j = 0; j < t.J; ++j) dd += (xs[j] - mean) * (xs[j] - mean);
    for (int j = 0; j < t.J; ++j) w[j] = (xs[j] - mean) / dd;
  }
  t.ln_len = need;
  for (int j = 0; j < t.J; ++j) {
    t.hw[j] = w[j];
    t.hqmax[j] = q[j * 256 + 255] - q[j * 256 + 0];
    for (int sh = 0; sh < 8 && t.qshift[j] < 0; ++sh) {
      bool ok = true;
      for (int v = 0; v < 256 && ok; ++v) ok = q[j * 256 + v] == (v >> sh);
      if (ok) t.qshift[j] = sh;
    }
  }
  // the tables depend only on (device, side, ln values, weights): upload once
  // and keep them (a few KB per block side) instead of copying every call
  static std::mutex mu;
  static std::map<std::vector<double>, DbcTables> cache;
  int dev = 0;
  FIC_CUDA(cudaGetDevice(&dev));
  std::vector<double> key{(double)dev, (double)side, (double)need, (double)gray_levels};
  key.insert(key.end(), w.begin(), w.end());
  key.insert(key.end(), ln.begin(), ln.end());
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  FIC_CUDA(cudaMalloc(&t.quot, t.J * 256 * sizeof(uint16_t)));
  FIC_CUDA(cudaMalloc(&t.ln, need * sizeof(double)));
  FIC_CUDA(cudaMalloc(&t.w, t.J * sizeof(double)));
  FIC_CUDA(cudaMemcpy(t.quot, q.data(), t.J * 256 * sizeof(uint16_t), cudaMemcpyHostToDevice));
  FIC_CUDA(cudaMemcpy(t.ln, ln.data(), need * sizeof(double), cudaMemcpyHostToDevice));
  FIC_CUDA(cudaMemcpy(t.w, w.data(), t.J * sizeof(double), cudaMemcpyHostToDevice));
  t.hln = new std::vector<double>(ln);
  cache.emplace(std::move(key), t);
  (void)sc;
  (void)s;
  return t;
}

// ---------------------------------------------------------------------------
// planning kernels
// ---------------------------------------------------------------------------
__global__ void k_iota(uint32_t* o, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = (uint32_t)i;
}

__global__ void k_bits_to_double(const unsigned long long* k, double* o, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = __longlong_as_double((long long)k[i]);
}

constexpr int kMaxRangeBins = 2 * (kCountSortMaxRanks + 1);

struct ClassifyArgs {
  const int32_t* lo;
  const int32_t* hi;
  int R;
  int n_iso;
  int small_pool;
  int tensor_ok;
  unsigned long long* key;     // (class << 63) | lo << 32 | hi
  uint32_t* rid;
  int64_t* pool_out;           // may be null
  unsigned long long* pool_sum;
  // optional counting-sort bins (rank form of the FD order): bin = class *
  // (n_rank + 1) + rank of lo, with the histogram of the bins
  const uint32_t* lo_rank;      // [R] rank index of lo (from k_slabs)
  int n_rank;
  uint32_t* bin;
  uint32_t* bin_hist;
};

__global__ void k_classify(ClassifyArgs a) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long pool = 0;
  if (r < a.R) {
    int32_t lo = a.lo[r], hi = a.hi[r];
    pool = (unsigned long long)(hi - lo);
    unsigned long long cls = (a.tensor_ok && (int64_t)pool >= a.small_pool) ? 0ull : 1ull;
    a.key[r] = (cls << 63) | ((unsigned long long)(uint32_t)lo << 32) | (uint32_t)hi;
    a.rid[r] = r;
    if (a.bin) {  // lo_rank orders like lo (rank_start is monotone)
      const uint32_t b = (uint32_t)cls * (uint32_t)(a.n_rank + 1) + a.lo_rank[r];
      a.bin[r] = b;
      // neighbouring ranges often share a bin: one atomic per group of equal bins
      const unsigned grp = __match_any_sync(__activemask(), b);
      if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(a.bin_hist + b, (uint32_t)__popc(grp));
    }
    if (a.pool_out) a.pool_out[r] = (int64_t)pool;
  }
  for (int m = 16; m >= 1; m >>= 1) pool += __shfl_xor_sync(0xffffffffu, pool, m);
  __shared__ unsigned long long wsum[32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = pool;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wsum[w];
    if (t) atomicAdd(a.pool_sum, t);
  }
}

__global__ void k_shard(const unsigned long long* key, const unsigned long long* cum, int R,
                        int shard, int nshard, PlanCounts* out) {
  if (threadIdx.x || blockIdx.x) return;
  // first position with class bit set
  int lo = 0, hi = R;
  while (lo < hi) {
    int m = (lo + hi) >> 1;
    if ((key[m] >> 63) == 0) lo = m + 1; else hi = m;
  }
  out->n_tensor = lo;
  // shard of position i: floor((cum[i] - 1) * nshard / total)
  unsigned long long total = R ? cum[R - 1] : 0;
  auto first_with_shard_ge = [&](int s) {
    int a = 0, b = R;
    while (a < b) {
      int m = (a + b) >> 1;
      unsigned long long sh = (cum[m] - 1) * (unsigned long long)nshard / total;
      if ((int)sh < s) a = m + 1; else b = m;
    }
    return a;
  };
  if (nshard <= 1 || total == 0) {
    out->shard_begin = 0;
    out->shard_end = R;
  } else {
    out->shard_begin = first_with_shard_ge(shard);
    out->shard_end = first_with_shard_ge(shard + 1);
  }
}

// Counting sort of the ranges by bin (class, rank of lo): the same grouping
// as the (class, lo) radix sort -- lo is a pure function of the rank -- in
// one scan block and one scatter pass.  Order inside a bin is unspecified;
// it only shapes the tiles, never the result.
__global__ void __launch_bounds__(1024) k_bin_scan(const uint32_t* hist, int nb, uint32_t* cursor,
                                                   int class1_bin, int R, PlanCounts* pc) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t s_carry;
  constexpr int IPT = 8;
  uint32_t carry = 0;
  for (int base = 0; base < nb; base += 1024 * IPT) {
    uint32_t v[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int b = base + threadIdx.x * IPT + i;
      v[i] = b < nb ? hist[b] : 0u;
    }
    uint32_t total = 0;
    Scan(tmp).ExclusiveSum(v, v, total);
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int b = base + threadIdx.x * IPT + i;
      if (b < nb) cursor[b] = carry + v[i];
      if (b == class1_bin) s_carry = carry + v[i];
    }
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // single shard: the whole sorted list, tensor class first
    pc->shard_begin = 0;
    pc->shard_end = R;
    pc->n_tensor = class1_bin < nb ? (int64_t)s_carry : R;
    pc->pool_sum = 0;
  }
}

__global__ void __launch_bounds__(1024) k_range_scatter(const uint32_t* bin, const unsigned long long* key,
                                                        int R, int nb, uint32_t* cursor,
                                                        unsigned long long* key_s, uint32_t* rid_s) {
  extern __shared__ uint32_t cnt[];  // [nb]
  constexpr int IPT = 4;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  const int r0 = blockIdx.x * blockDim.x * IPT;
  uint32_t bb[IPT], loc[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int r = r0 + i * blockDim.x + threadIdx.x;
    bb[i] = r < R ? bin[r] : 0u;
    if (r < R) loc[i] = atomicAdd(cnt + bb[i], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (cnt[b]) cnt[b] = atomicAdd(cursor + b, cnt[b]);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int r = r0 + i * blockDim.x + threadIdx.x;
    if (r < R) {
      const uint32_t pos = cnt[bb[i]] + loc[i];
      key_s[pos] = key[r];
      rid_s[pos] = (uint32_t)r;
    }
  }
}

// Stable, deterministic variant of the counting sort (sharded calls: every
// rank must cut the same order, so ties inside a bin keep raster order).
// Ranges are cut into chunks of kStableChunk; k_chunk_hist counts the bins of
// each chunk into a bin-major [nb][nchunk] matrix, whose exclusive scan
// (k_bin_scan) is each (bin, chunk)'s first output position; one warp per
// chunk then places its ranges in order (__match_any_sync ranks equal bins
// within a round of 32, a shared counter per bin carries across rounds).
constexpr int kStableChunk = 2048;

__global__ void __launch_bounds__(1024) k_chunk_hist(const uint32_t* bin, int R, int nb,
                                                     int nchunk, uint32_t* mat) {
  extern __shared__ uint32_t cnt[];  // [nb]
  for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  const int r0 = blockIdx.x * kStableChunk;
  for (int i = threadIdx.x; i < kStableChunk; i += blockDim.x)
    if (r0 + i < R) atomicAdd(cnt + bin[r0 + i], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) mat[(int64_t)b * nchunk + blockIdx.x] = cnt[b];
}

__global__ void __launch_bounds__(32) k_range_scatter_stable(const uint32_t* bin,
                                                             const unsigned long long* key, int R,
                                                             int nb, int nchunk,
                                                             const uint32_t* start,
                                                             unsigned long long* key_s,
                                                             uint32_t* rid_s) {
  extern __shared__ uint32_t cur[];  // [nb] next position of each bin in this chunk
  const int lane = threadIdx.x;
  for (int b = lane; b < nb; b += 32) cur[b] = start[(int64_t)b * nchunk + blockIdx.x];
  __syncwarp();
  const int r0 = blockIdx.x * kStableChunk, r1 = min(R, r0 + kStableChunk);
  for (int base = r0; base < r1; base += 32) {
    const int r = base + lane;
    const bool ok = r < r1;
    const uint32_t b = ok ? bin[r] : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    uint32_t pos = 0;
    if (ok) pos = cur[b] + rank;
    __syncwarp();
    if (ok && rank == 0) cur[b] += __popc(peers);
    __syncwarp();
    if (ok) {
      key_s[pos] = key[r];
      rid_s[pos] = (uint32_t)r;
    }
  }
}

// Inclusive scan of the per-position shard costs (one block; k_cost's rule).
__global__ void __launch_bounds__(1024) k_cost_scan(const unsigned long long* key, int R,
                                                    int n_iso, unsigned long long* cum) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  unsigned long long carry = 0;
  for (int base = 0; base < R; base += 1024 * 4) {
    unsigned long long v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = base + threadIdx.x * 4 + i;
      v[i] = 0;
      if (k < R) {
        const unsigned long long kk = key[k];
        const unsigned long long pool = (uint32_t)kk - (uint32_t)((kk >> 32) & 0x7fffffffu);
        // an exact-path candidate costs ~32x a screened one (as k_cost);
        // every range also carries its share of a tensor tile's fixed cost
        // (item setup, pipeline fill: ~0.7 us per 16-range tile at cfg3 =
        // ~3.5e5 screened candidates per range), or the shard of the
        // small-window ranges at the end of the order runs long
        v[i] = pool * n_iso * ((kk >> 63) ? 32ull : 1ull) + (1ull << 18);
      }
    }
    unsigned long long t = 0;
    Scan(tmp).InclusiveSum(v, v, t);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = base + threadIdx.x * 4 + i;
      if (k < R) cum[k] = carry + v[i];
    }
    carry += t;
    __syncthreads();
  }
}

// tensor / exact positions of this shard in the sorted range list
struct PlanRange {
  int64_t tb, te, eb, ee;
};
__device__ __forceinline__ PlanRange plan_range(const PlanCounts* pc) {
  PlanRange q;
  q.tb = pc->shard_begin;
  q.te = max(q.tb, min(pc->shard_end, pc->n_tensor));
  q.eb = max(pc->shard_begin, pc->n_tensor);
  q.ee = max(q.eb, pc->shard_end);
  return q;
}

struct TileArgs {
  const unsigned long long* key;  // sorted
  const uint32_t* rid;            // sorted
  const PlanCounts* pc;           // tensor positions of this shard (device)
  int RT;
  int seg;
  int seg0;
  int32_t* wlo;
  int32_t* whi;
  int32_t* nseg;
  int32_t* nslots;                // [R]
  int n_iso;
  unsigned long long* useful;     // sum(pool) * n_iso over tensor ranges
  int nsub;                       // partial slots per segment (tail splitting, TcArgs::nsub)
};

__global__ void k_tiles(TileArgs a) {
  const PlanRange q = plan_range(a.pc);
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t b = q.tb + t * a.RT;
  if (b >= q.te) return;
  int64_t e = min(q.te, b + a.RT);
  int32_t lo = (int32_t)((a.key[b] >> 32) & 0x7fffffffu);
  int32_t hi = 0;
  for (int64_t i = b; i < e; ++i) hi = max(hi, (int32_t)(uint32_t)a.key[i]);
  // a short first segment (seg0 columns), then seg-column segments
  int32_t ns = (hi <= lo) ? 0 : (hi - lo <= a.seg0) ? 1 : 1 + (int32_t)cdiv(hi - lo - a.seg0, a.seg);
  a.wlo[t] = lo;
  a.whi[t] = hi;
  a.nseg[t] = ns;
  unsigned long long u = 0;
  for (int64_t i = b; i < e; ++i) {
    a.nslots[a.rid[i]] = ns * a.nsub;
    unsigned long long k = a.key[i];
    u += (uint32_t)k - (uint32_t)((k >> 32) & 0x7fffffffu);
  }
  atomicAdd(a.useful, u * a.n_iso);
  atomicAdd(a.useful - 2, (unsigned long long)(hi - lo) * (unsigned long long)((e - b) * a.n_iso));
}

__global__ void k_exact_segs(const unsigned long long* key, const uint32_t* rid, const PlanCounts* pc,
                             int seg, int32_t* nseg, int32_t* nslots) {
  const PlanRange q = plan_range(pc);
  const int64_t eb = q.eb, ee = q.ee;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (eb + i >= ee) return;
  unsigned long long k = key[eb + i];
  int32_t pool = (int32_t)((uint32_t)k - (uint32_t)((k >> 32) & 0x7fffffffu));
  int32_t ns = (int32_t)cdiv(pool, seg);
  nseg[i] = ns;
  nslots[rid[eb + i]] = ns;
}

// Exclusive scans of the per-tile and per-exact-range segment counts and of
// the per-range slot counts (int64), plus their totals, in one block.
template <class T, class U>
__device__ void block_exclusive_scan(const T* in, U* out, int64_t n, U* total) {
  using Scan = cub::BlockScan<U, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  U carry = 0;
  for (int64_t base = 0; base < n; base += 1024 * 4) {
    U v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t k = base + threadIdx.x * 4 + i;
      v[i] = k < n ? (U)in[k] : (U)0;
    }
    U t = 0;
    Scan(tmp).ExclusiveSum(v, v, t);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t k = base + threadIdx.x * 4 + i;
      if (k < n) out[k] = carry + v[i];
    }
    carry += t;
    __syncthreads();
  }
  *total = carry;
}

// ... and the device-side plan (DevPlan) the matchers read their counts from.
__global__ void __launch_bounds__(1024) k_plan_scans(const int32_t* tnseg, int32_t* tbase,
                                                     const int32_t* enseg, int32_t* ebase,
                                                     const int32_t* nslots, int64_t* sbase, int R,
                                                     const PlanCounts* pc, int RT, int nsub,
                                                     int split_cap, DevPlan* dp) {
  const PlanRange q = plan_range(pc);
  const int64_t n_tr = q.te - q.tb, n_er = q.ee - q.eb, ntt = cdiv(n_tr, RT);
  // three independent scans, one block each
  if (blockIdx.x == 0) {
    int32_t t = 0;
    block_exclusive_scan<int32_t, int32_t>(tnseg, tbase, ntt, &t);
    if (threadIdx.x == 0) {
      dp->tb = q.tb;
      dp->n_tr = n_tr;
      dp->n_tt = ntt;
      dp->n_titems = t;
      dp->n_split = nsub > 1 ? min((int64_t)t, (int64_t)split_cap) : 0;
    }
  } else if (blockIdx.x == 1) {
    int32_t t = 0;
    block_exclusive_scan<int32_t, int32_t>(enseg, ebase, n_er, &t);
    if (threadIdx.x == 0) {
      dp->eb = q.eb;
      dp->n_er = n_er;
      dp->n_eitems = t;
    }
  } else {
    int64_t t = 0;
    block_exclusive_scan<int32_t, int64_t>(nslots, sbase, R, &t);
    if (threadIdx.x == 0) dp->n_slots = t;
  }
}


__global__ void k_expand(const int32_t* nseg, const int32_t* base, const DevPlan* dp, int2* items) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= dp->n_er) return;
  int32_t b = base[t];
  for (int s = 0; s < nseg[t]; ++s) items[b + s] = make_int2((int)t, s);
}

// Work items in segment-major order: every tile's segment s before any
// segment s + 1, so later segments start from the thresholds the earlier
// ones found, and inside a segment in tile order, so the items running
// together read neighbouring FD windows (L2 reuse).  k_seg_hist counts the
// tiles per segment count, k_seg_base turns that into each segment's first
// item, k_seg_place places each segment's items (one block per segment).
__global__ void k_seg_hist(const int32_t* nseg, const DevPlan* dp, int smax, uint32_t* hist) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= dp->n_tt) return;
  atomicAdd(hist + min((int)nseg[t], smax), 1u);
}

__global__ void __launch_bounds__(1024) k_seg_base(const uint32_t* hist, int smax, uint32_t* base,
                                                   uint32_t* cursor) {
  // cnt[s] = tiles with more than s segments; base = exclusive scan of cnt
  if (threadIdx.x != 0) return;
  uint32_t above = 0, acc = 0;
  for (int v = smax; v >= 1; --v) {  // cnt[v - 1] = sum of hist[v .. smax]
    above += hist[v];
    cursor[v - 1] = above;           // temporarily the count
  }
  for (int s2 = 0; s2 < smax; ++s2) {
    const uint32_t c = cursor[s2];
    base[s2] = acc;
    acc += c;
    cursor[s2] = 0;
  }
}

// Segment s's items in tile order: block s scans the flags (tile t has a
// segment s) and places (t, s) at base[s] + its rank -- the (segment, tile)
// order of the round-1 single-block loop, in parallel over the segments.
__global__ void __launch_bounds__(1024) k_seg_place(const int32_t* nseg, const DevPlan* dp,
                                                    const uint32_t* base, int2* items) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const int sg = blockIdx.x;
  const int64_t n = dp->n_tt;
  int64_t carry = base[sg];
  for (int64_t t0 = 0; t0 < n; t0 += 1024) {
    const int64_t t = t0 + threadIdx.x;
    const int flag = (t < n && nseg[t] > sg) ? 1 : 0;
    int rank = 0, total = 0;
    Scan(tmp).ExclusiveSum(flag, rank, total);
    if (flag) items[carry + rank] = make_int2((int)t, sg);
    carry += total;
    __syncthreads();
  }
}

// ---- compact FD sort ---------------------------------------------------
// With a few scales and small counts the domain FDs take few distinct values
// (side 16: FD depends on (N2, N8) only, the middle weight being 0.0), so the
// stable sort by FD becomes a stable sort by the rank of the value among all
// possible values: same order, ~12-bit keys instead of 52-bit ones.  The
// rank table depends only on the DBC tables, so the host builds it once (the
// same fp64 op sequence as the kernels: product, then left-to-right sum,
// clamp) and keeps it on the device.
struct FdCombo {
  int J, C;                 // scales, number of combinations
  int k2[7], cstride[7], crange[7];  // cells per block, index stride / range (0 = inactive)
};
struct RankTable {
  uint32_t* rank_of_combo = nullptr;  // [C]
  double* fd_of_rank = nullptr;       // [n_rank] strictly increasing
  int n_rank = 0;
};

static RankTable make_rank_table(const DbcTables& td, const FdCombo& fc, int clamp) {
  static std::mutex mu;
  static std::map<std::vector<int64_t>, RankTable> cache;
  int dev = 0;
  FIC_CUDA(cudaGetDevice(&dev));
  std::vector<int64_t> key{dev, (int64_t)(uintptr_t)td.quot, fc.J, fc.C, clamp};
  for (int j = 0; j < fc.J; ++j) {
    key.push_back(fc.k2[j]);
    key.push_back(fc.cstride[j]);
    key.push_back(fc.crange[j]);
  }
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const std::vector<double>& ln = *td.hln;
  std::vector<double> val(fc.C);
  for (int c = 0; c < fc.C; ++c) {
    double f = 0.0;
    for (int j = 0; j < fc.J; ++j) {  // k_fd: __dmul_rn then __dadd_rn, no contraction
      const int raw = fc.cstride[j] ? (c / fc.cstride[j]) % fc.crange[j] : 0;
      const int cnt = std::min(raw + fc.k2[j], td.ln_len - 1);
      volatile double t = ln[cnt] * td.hw[j];
      f = (j == 0) ? (double)t : f + (double)t;
    }
    if (clamp) f = std::fmin(std::fmax(f, 2.0), 3.0);
    val[c] = f;
  }
  std::vector<int> idx(fc.C);
  for (int c = 0; c < fc.C; ++c) idx[c] = c;
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return val[x] < val[y]; });
  std::vector<uint32_t> rank(fc.C);
  std::vector<double> fdr;
  for (int i = 0; i < fc.C; ++i) {
    if (i == 0 || val[idx[i]] != val[idx[i - 1]]) fdr.push_back(val[idx[i]]);
    rank[idx[i]] = (uint32_t)(fdr.size() - 1);
  }
  RankTable rt;
  rt.n_rank = (int)fdr.size();
  FIC_CUDA(cudaMalloc(&rt.rank_of_combo, fc.C * sizeof(uint32_t)));
  FIC_CUDA(cudaMalloc(&rt.fd_of_rank, fdr.size() * sizeof(double)));
  FIC_CUDA(cudaMemcpy(rt.rank_of_combo, rank.data(), fc.C * sizeof(uint32_t), cudaMemcpyHostToDevice));
  FIC_CUDA(cudaMemcpy(rt.fd_of_rank, fdr.data(), fdr.size() * sizeof(double), cudaMemcpyHostToDevice));
  cache.emplace(std::move(key), rt);
  return rt;
}

__global__ void k_sl_init(unsigned long long* best, unsigned long long* pre, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  best[2 * i] = ~0ull;
  best[2 * i + 1] = ord_bits(INFINITY);
  pre[i] = ord_bits(INFINITY);
}

__global__ void k_fill_u64(unsigned long long* a, unsigned long long v, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
__global__ void k_i32_to_i64(const int32_t* a, int64_t* o, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i];
}
__global__ void k_u32_to_i64(const uint32_t* a, int64_t* o, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i];
}

// CUB helpers (temp storage from the scratch pool)
template <class F>
static void cub_call(Scratch& sc, F f) {
  size_t bytes = 0;
  FIC_CUDA(f(nullptr, bytes));
  void* tmp = sc.get<uint8_t>(bytes);
  FIC_CUDA(f(tmp, bytes));
}

// ---------------------------------------------------------------------------
// pool planning shared by encode and plan
// ---------------------------------------------------------------------------
struct PlanBufs {
  const uint32_t* rank_start = nullptr;  // [n_rank + 1] rank form of the FD order (else null)
  int n_rank = 0;
  const uint32_t* lo_rank = nullptr;     // [R] rank index of each slab start (dynamic_fd, rank form)
  double* fd_dom = nullptr;      // [D] (dynamic/static2)
  double* fd_rng = nullptr;      // [R]
  double* keys = nullptr;        // [D] sorted FDs
  uint32_t* order = nullptr;     // [D] raster id per pool position (nullptr = identity)
  int32_t* lo = nullptr;
  int32_t* hi = nullptr;
  double* scal = nullptr;        // [4]
};

static PlanBufs make_plan(Scratch& sc, cudaStream_t s, const uint8_t* img, const Geo& g,
                          const fic_params_t& p, bool want_fd_dom, bool stable_order,
                          double* scal_buf = nullptr) {
  PlanBufs pb;
  pb.lo = sc.get<int32_t>(g.R);
  pb.hi = sc.get<int32_t>(g.R);
  pb.scal = scal_buf ? scal_buf : sc.get<double>(4);
  FIC_CUDA(cudaMemsetAsync(pb.scal, 0, 4 * sizeof(double), s));
  SlabArgs sa{};
  sa.R = g.R;
  sa.D = g.D;
  sa.strategy = p.strategy;
  sa.has_delta = p.has_delta;
  sa.delta = p.delta;
  sa.scal = pb.scal;
  sa.lo = pb.lo;
  sa.hi = pb.hi;
  sa.H = g.H;
  sa.W = g.W;
  sa.rs = g.rs;
  sa.ds = g.ds;
  sa.st = g.st;
  sa.nrx = g.nrx;
  sa.ndx = g.ndx;
  if (p.strategy == FIC_STATIC2 || p.strategy == FIC_DYNAMIC_FD) {
    // K2: FD of domains (original or decimated blocks) then ranges, in the
    // reference's order so the same side raises first (codec.py:352-354)
    int dside = p.fd_source == FIC_FD_ORIGINAL ? g.ds : g.rs;
    DbcTables td = make_dbc(sc, s, dside, p.h_ln_table, p.ln_len, p.h_fd_weights_dom,
                            p.n_fd_weights_dom);
    DbcTables tr = make_dbc(sc, s, g.rs, p.h_ln_table, p.ln_len, p.h_fd_weights_rng,
                            p.n_fd_weights_rng);
    pb.fd_dom = want_fd_dom ? sc.get<double>(g.D) : nullptr;
    pb.fd_rng = sc.get<double>(g.R);
    uint32_t* iin = sc.get<uint32_t>(g.D);
    pb.order = sc.get<uint32_t>(g.D);
    FdArgs fa{};
    fa.src = img;
    fa.W = g.W;
    fa.side = dside;
    fa.bst = g.st;
    fa.nbx = g.ndx;
    fa.n = g.D;
    fa.mode = p.fd_source == FIC_FD_ORIGINAL ? FD_IMAGE : FD_DECIMATED;
    fa.clamp = 1;
    fa.J = td.J;
    fa.smax = td.smax;
    fa.quot = td.quot;
    fa.ln = td.ln;
    fa.ln_len = td.ln_len;
    fa.w = td.w;
    for (int j = 0; j < 7; ++j) fa.qshift[j] = td.qshift[j];
    fa.fd = pb.fd_dom;
    // compact-key path: enumerate the count combinations of the scales with
    // a nonzero weight (a zero weight adds +0.0 whatever the count)
    FdCombo fc{};
    fc.J = td.J;
    fc.C = 1;
    for (int j = 0; j < td.J; ++j) {
      const int kk = dside >> (j + 1);
      fc.k2[j] = kk * kk;
      const int64_t range = (int64_t)kk * kk * td.hqmax[j] + 1;
      if (td.hw[j] != 0.0 && fc.C * range <= 65536) {
        fc.cstride[j] = fc.C;
        fc.crange[j] = (int)range;
        fc.C *= (int)range;
      } else if (td.hw[j] != 0.0) {
        fc.C = 0;  // too many values: fall back to the 52-bit sort
        break;
      }
    }
    const bool compact = fc.C > 0 && fa.clamp && dside <= 16 && (td.smax == 4 || td.smax == 8) &&
                         !getenv("FIC_FD_WIDE_SORT");
    RankTable rt;
    uint32_t* rk = nullptr;
    unsigned long long* kin = nullptr;
    uint32_t* hist = nullptr;
    bool count_sort = false;
    if (compact) {
      rt = make_rank_table(td, fc, fa.clamp);
      rk = sc.get<uint32_t>(g.D);
      fa.rank_of_combo = rt.rank_of_combo;
      fa.rank = rk;
      for (int j = 0; j < td.J; ++j) fa.cstride[j] = fc.cstride[j];
      // encode does not need the reference's order among equal FDs (see
      // k_rank_scatter); plan() returns it, so it keeps the stable sort
      count_sort = !stable_order && rt.n_rank <= kCountSortMaxRanks && !getenv("FIC_FD_STABLE");
      if (count_sort) {
        hist = sc.get<uint32_t>(2 * rt.n_rank);
        FIC_CUDA(cudaMemsetAsync(hist, 0, rt.n_rank * sizeof(uint32_t), s));
        FIC_CUDA(cudaMemsetAsync(hist + rt.n_rank, 0xff, rt.n_rank * sizeof(uint32_t), s));
        fa.rank_hist = hist;
        fa.rank_minid = hist + rt.n_rank;
        fa.n_rank = rt.n_rank;
      }
    } else {
      kin = sc.get<unsigned long long>(g.D);
      fa.key = kin;
    }
    fa.iota = count_sort ? nullptr : iin;
    launch_fd(fa, s);
    FdArgs fr{};
    fr.src = img;
    fr.W = g.W;
    fr.side = g.rs;
    fr.bst = g.rs;
    fr.nbx = g.nrx;
    fr.n = g.R;
    fr.mode = FD_IMAGE;
    fr.clamp = 1;
    fr.J = tr.J;
    fr.smax = tr.smax;
    fr.quot = tr.quot;
    fr.ln = tr.ln;
    fr.ln_len = tr.ln_len;
    fr.w = tr.w;
    fr.fd = pb.fd_rng;
    launch_fd(fr, s);
    // K3: stable sort of domains by FD (== AvlTree flatten, avltree.py:150-189)
    if (compact) {
      uint32_t* rstart = sc.get<uint32_t>(rt.n_rank + 1);
      if (count_sort) {
        uint32_t* cursor = sc.get<uint32_t>(rt.n_rank);
        ScalArgs scl{rt.fd_of_rank, p.strategy, p.has_delta, p.delta, pb.scal};
        launch_count_sort(rk, g.D, rt.n_rank, hist, hist + rt.n_rank, rstart, cursor, pb.order, scl,
                          s);
        sa.scal_ready = 1;
      } else {
        // stable sort of the domains by rank (same order as by FD value)
        uint32_t* rks = sc.get<uint32_t>(g.D);
        int rbits = 1;
        while ((1 << rbits) < rt.n_rank) ++rbits;
        cub_call(sc, [&](void* t, size_t& b) {
          return cub::DeviceRadixSort::SortPairs(t, b, rk, rks, iin, pb.order, (int64_t)g.D, 0,
                                                 rbits, s);
        });
        launch_rank_start(rks, g.D, rt.n_rank, rstart, s);
      }
      sa.keys = nullptr;
      pb.rank_start = rstart;
      pb.n_rank = rt.n_rank;
      if (p.strategy == FIC_DYNAMIC_FD) {
        uint32_t* lr = sc.get<uint32_t>(g.R);
        sa.lo_rank = lr;
        pb.lo_rank = lr;
      }
      sa.fd_of_rank = rt.fd_of_rank;
      sa.rank_start = rstart;
      sa.n_rank = rt.n_rank;
    } else {
      // FDs are clamped to [2, 3] (fa.clamp), so the sign and exponent bits of
      // every key are equal (0x400): sorting the 52 mantissa bits is exact
      unsigned long long* kout = sc.get<unsigned long long>(g.D);
      const int nbits = fa.clamp ? 52 : 64;
      cub_call(sc, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, iin, pb.order, (int64_t)g.D, 0,
                                               nbits, s);
      });
      pb.keys = sc.get<double>(g.D);
      k_bits_to_double<<<(unsigned)cdiv(g.D, 256), 256, 0, s>>>(kout, pb.keys, g.D);
      FIC_CHECK_LAUNCH();
      sa.keys = pb.keys;
    }
    sa.ids = pb.order;
    sa.fd_rng = pb.fd_rng;
  }
  launch_slabs(sa, s);
  return pb;
}

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

template <class F>
static int guarded(F f) {
  try {
    f();
    return FIC_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return FIC_ECUDA;
  }
}

// ---------------------------------------------------------------------------
// encode
// ---------------------------------------------------------------------------
// Inverse isometry tables (blocks.py:113-139) on the device, built and
// uploaded once per (device, range size): a per-call pageable copy would make
// the host wait for the work already queued on the stream.
static const int* iso_inverse_table(int dev, int rs) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, int*> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, rs});
  if (it != cache.end()) return it->second;
  const int K = rs * rs;
  std::vector<int> perm(8 * K), inv(8 * K);
  iso_tables(rs, perm.data(), inv.data());
  int* d = nullptr;
  FIC_CUDA(cudaMalloc(&d, 8 * K * sizeof(int)));
  FIC_CUDA(cudaMemcpy(d, inv.data(), 8 * K * sizeof(int), cudaMemcpyHostToDevice));
  cache.emplace(std::make_pair(dev, rs), d);
  return d;
}

// K1 buffers: what the matchers read per pool position (fp16 B rows on the
// tensor path, sums, 1/den) plus the source of the decimated pixels -- the
// row segments or box-floor planes the builder stages anyway (8x8 / 4x4
// ranges), or a zero-padded raw copy for other range sizes.
static PoolArgs pool_args(Scratch& sc, const Geo& g, const uint8_t* img, const uint32_t* order,
                          bool tensor_ok) {
  PoolArgs pa{};
  pa.img = img;
  pa.H = g.H;
  pa.W = g.W;
  pa.rs = g.rs;
  pa.plane_rows = g.H - 1;
  pa.pitch = (int)align_up((size_t)(g.W / 2 + 16), 16);
  pa.mh = g.H / 2;
  pa.KP = (int)align_up((size_t)g.npx, 4);
  // 8x8 ranges: per-domain-column row segments when they fit well inside L2
  // (cfg3: 8.3 MB), else the box-floor planes (cfg5: T would be 268 MB)
  const size_t t_bytes = (size_t)g.ndx * 2 * pa.mh * 8;
  if (g.rs == 8 && g.st <= 16 && t_bytes <= ((size_t)48 << 20) && !getenv("FIC_POOL_PLANES"))
    pa.trows = sc.get<unsigned long long>(t_bytes / 8);
  else if (g.rs == 8 || g.rs == 4)
    pa.planes = sc.get<uint8_t>((size_t)2 * pa.plane_rows * pa.pitch + 16);
  else
    pa.raw = sc.get<uint8_t>((size_t)g.D * pa.KP);
  pa.st = g.st;
  pa.ndx = g.ndx;
  pa.D = g.D;
  pa.order = order;
  pa.bh = tensor_ok ? sc.get<uint16_t>((size_t)g.D * g.npx) : nullptr;
  pa.inv_den = sc.get<double>(g.D);
  pa.sums = sc.get<uint2>(g.D);
  return pa;
}

static PoolView pool_view(const PoolArgs& pa) {
  PoolView P{};
  P.bh = pa.bh;
  P.inv_den = pa.inv_den;
  P.sums = pa.sums;
  P.order = pa.order;
  P.D = pa.D;
  P.src.trows = pa.trows;
  P.src.planes = pa.planes;
  P.src.raw = pa.raw;
  P.src.ndx = pa.ndx;
  P.src.st = pa.st;
  P.src.mh = pa.mh;
  P.src.plane_rows = pa.plane_rows;
  P.src.pitch = pa.pitch;
  P.src.KP = pa.KP;
  return P;
}

// Everything an encode reads back at the end, in one block (one copy).
struct Readback {
  unsigned long long counters[16];
  double scal[4];
  DevPlan plan;
  unsigned long long flat[2];  // [0] flat count, [1] low word: canonical flat range
  uint32_t sl_count[4];        // [0] survivor-list entries appended, [1] hit-list entries, [2] sorted
  unsigned long long hl_tests;  // hit-list lower-bound tests
};

// Pinned host copy of the readback (per thread, device and stream): the
// copy is then part of a captured graph.
static Readback* pinned_readback(int dev, cudaStream_t s) {
  static thread_local std::map<std::pair<int, cudaStream_t>, Readback*> m;
  Readback*& p = m[{dev, s}];
  if (!p) FIC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), sizeof(Readback), cudaHostAllocDefault));
  return p;
}

// Host state the part of an encode after the readback needs.
struct EncPost {
  bool flat_path = false;
  FlatArgs fl{};
  PoolView P{};
  const int32_t* lo = nullptr;
  const int32_t* hi = nullptr;
  int32_t* nslots = nullptr;
  uint32_t sl_cap = 0, hl_cap = 0;
  int launches = 0;
  size_t sc_off = 0;
};

// CUDA graphs of whole encodes.  A call's device work (about 25 launches,
// memsets, the side-stream fork / join and the readback copy) depends only
// on its arguments and on the arena addresses, so a call that repeats a
// previous one exactly -- same device, stream, image and output pointers,
// parameters and arena -- is recorded as a graph on its second occurrence
// and replayed from then on: one launch instead of the host enqueueing
// every kernel while the GPU waits on the short planning kernels.  Calls
// with any FIC_* experiment variable set, or whose arena is still growing,
// run directly; a failed capture falls back to the direct path.
struct GraphKey {
  std::vector<int64_t> v;
  bool operator<(const GraphKey& o) const { return v < o.v; }
};
struct GraphEnt {
  cudaGraphExec_t exec = nullptr;
  EncPost post;
};
thread_local bool g_capturing = false;
static thread_local std::map<GraphKey, GraphEnt> g_graphs;
static thread_local std::set<GraphKey> g_graph_seen;

static bool graphs_allowed() {
  for (char** e = ::environ; e && *e; ++e)
    if (std::strncmp(*e, "FIC_", 4) == 0) return false;
  return true;
}

// The stream graphs are recorded and replayed on (per thread and device):
// the caller's stream may be the legacy default stream, which cannot be
// captured; events order it after the caller's stream and back.
struct GraphStream {
  cudaStream_t gs = nullptr;
  cudaEvent_t in = nullptr, out = nullptr;
  static GraphStream& get(int dev) {
    static thread_local std::map<int, GraphStream> m;
    GraphStream& g = m[dev];
    if (!g.gs) {
      FIC_CUDA(cudaStreamCreateWithFlags(&g.gs, cudaStreamNonBlocking));
      FIC_CUDA(cudaEventCreateWithFlags(&g.in, cudaEventDisableTiming));
      FIC_CUDA(cudaEventCreateWithFlags(&g.out, cudaEventDisableTiming));
    }
    return g;
  }
};
static thread_local bool g_graphs_off = false;  // a capture left a stream in a bad state

static void encode_impl(const uint8_t* img, int H, int W, const fic_params_t& p, uint8_t* records,
                        double* pre_rms, double* post_rms, int64_t* pool_sizes,
                        fic_stats_t* st, cudaStream_t s_user) {
  cudaStream_t s = s_user;  // the enqueue stream (the graph stream while recording / replaying)
  Geo g = validate(H, W, p);
  if (p.strategy == FIC_STATIC2 || p.strategy == FIC_DYNAMIC_FD) {
    check_dbc_side(p.fd_source == FIC_FD_ORIGINAL ? g.ds : g.rs);
    check_dbc_side(g.rs);
  }
  const int K = g.npx;
  const int nshard = std::max(1, p.shard_count);
  const int shard = std::min(std::max(0, p.shard_index), nshard - 1);
  // Small jobs (at most kSmallJob candidates even if every pool were the
  // whole domain set) go to the exact CUDA-core matcher: the tensor
  // pipeline's fixed cost (persistent grid, TMEM allocation, ring fill)
  // exceeds their work (cfg1: 0.285 -> 0.20 ms).  An explicit small_pool
  // keeps the caller's routing.
  constexpr int64_t kSmallJob = 16 << 20;
  const bool small_job = p.small_pool == 0 && (int64_t)g.R * g.D * g.n_iso <= kSmallJob;
  const bool tensor_ok = (p.matcher != FIC_MATCH_EXACT) && tc_supported(K) && !small_job;
  const int small_pool = p.small_pool > 0 ? p.small_pool : 256;
  const int seg_t = p.max_segment > 0 ? (int)align_up(p.max_segment, 256) : 131072;
  // first segment of each tensor tile (a multiple of the 128-column N-tile);
  // a short one seeds thresholds early but measured no faster at cfg3
  const int seg0 = getenv("FIC_SEG0") ? std::max(128, atoi(getenv("FIC_SEG0")) / 128 * 128) : seg_t;
  const int seg_e = 4096;
  // tail splitting of the tensor work items (TcArgs::nsub); FIC_TC_SPLIT=1 disables
  const int nsub = getenv("FIC_TC_SPLIT") ? std::max(1, atoi(getenv("FIC_TC_SPLIT"))) : 4;
  const int RT = (tensor_ok ? tc_tile_rows(K) : 128) / g.n_iso;

  g_launches = 0;
  Scratch sc(s);
  Timer tm(s);
  // FIC_PLAN_TIMING: extra events inside the planning phase (events 8..)
  const bool ptime = getenv("FIC_PLAN_TIMING") != nullptr;
  int pn = 8;
  auto pmark = [&]() {
    if (ptime && pn < 21) FIC_CUDA(cudaEventRecord(tm.ev[pn++], s));
  };
  SideStream& side = SideStream::get();
  int dev_id = 0;
  FIC_CUDA(cudaGetDevice(&dev_id));
  Readback* h_rb = pinned_readback(dev_id, s);

  // ---- the call's device work: enqueued directly, or recorded once as a
  // CUDA graph and replayed (g_graphs) ----
  auto enqueue = [&]() -> EncPost {
  EncPost post{};
  tm.n = 0;
  tm.mark();  // 0

  // flat ranges (fic_flat.cu): detected up front, counted at the first sync
  FlatArgs fl{};
  const bool flat_path = p.strategy != FIC_NOSEARCH && !getenv("FIC_NO_FLAT");
  Readback* d_rb = sc.get<Readback>(1);
  FIC_CUDA(cudaMemsetAsync(d_rb, 0, sizeof(Readback), s));
  unsigned long long* flat_ctr = d_rb->flat;
  if (flat_path) {
    fl.img = img;
    fl.W = g.W;
    fl.rs = g.rs;
    fl.nrx = g.nrx;
    fl.R = g.R;
    fl.K = K;
    fl.D = g.D;
    fl.flat_c = sc.get<int16_t>(g.R);
    fl.n_flat = flat_ctr;
    fl.canon = reinterpret_cast<uint32_t*>(flat_ctr + 1);
    FIC_CUDA(cudaMemsetAsync(flat_ctr + 1, 0xff, 8, s));
    launch_flat_detect(fl, s);
  }

  // ranges (side stream: needs only the image)
  const int* d_inv = iso_inverse_table(dev_id, g.rs);
  RangeArgs ra{};
  ra.img = img;
  ra.W = g.W;
  ra.rs = g.rs;
  ra.nrx = g.nrx;
  ra.R = g.R;
  ra.n_iso = g.n_iso;
  ra.inv_perm = d_inv;
  ra.info = sc.get<RangeInfo>(g.R);
  ra.KP = (int)align_up((size_t)K, 4);
  ra.rows = sc.get<uint8_t>((size_t)g.R * g.n_iso * ra.KP);
  // FIC_POOL_SERIAL: the side-stream work (range preparation, pool builder)
  // on the caller's stream -- a measurement of K1 with nothing beside it
  const bool pool_serial = getenv("FIC_POOL_SERIAL") != nullptr;
  FIC_CUDA(cudaEventRecord(side.ev[0], s));
  FIC_CUDA(cudaStreamWaitEvent(side.s2, side.ev[0], 0));
  launch_ranges(ra, pool_serial ? s : side.s2);

  PlanBufs pb = make_plan(sc, s, img, g, p, false, false, d_rb->scal);
  tm.mark();  // 1

  // K1 pool builder (side stream: needs the FD order, overlaps the planning)
  PoolArgs pa = pool_args(sc, g, img, pb.order, tensor_ok);
  cudaStream_t ps = pool_serial ? s : side.s2;
  pa.ev_main = side.ev[5];
  FIC_CUDA(cudaEventRecord(side.ev[1], s));
  FIC_CUDA(cudaStreamWaitEvent(side.s2, side.ev[1], 0));
  FIC_CUDA(record_timing_event(side.ev[3], ps));
  launch_pool(pa, ps);
  FIC_CUDA(record_timing_event(side.ev[4], ps));
  FIC_CUDA(cudaEventRecord(side.ev[2], side.s2));
  tm.mark();  // 2
  pmark();  // 8
  pmark();  // 9

  // plan: classify, sort by (class, lo, hi), shard by cost
  unsigned long long* counters = d_rb->counters;  // zeroed with the readback block
  unsigned long long* key = sc.get<unsigned long long>(g.R);
  unsigned long long* key_s = sc.get<unsigned long long>(g.R);
  uint32_t* rid = sc.get<uint32_t>(g.R);
  uint32_t* rid_s = sc.get<uint32_t>(g.R);
  ClassifyArgs ca{pb.lo, pb.hi, g.R, g.n_iso, small_pool, tensor_ok ? 1 : 0, key, rid,
                  pool_sizes, counters + 2};
  // counting sort by (class, rank of lo) when the FD order is in rank form
  const int nb = pb.rank_start ? 2 * (pb.n_rank + 1) : 0;
  // (the shard partition is a cut of this order: every rank must compute the
  // same one, so shards keep the deterministic stable radix sort)
  const bool bin_ok = pb.lo_rank && nb <= kMaxRangeBins && !getenv("FIC_RANGE_RADIX");
  const bool bin_sort = bin_ok && nshard == 1 && !getenv("FIC_RANGE_STABLE");
  const bool stable_sort = bin_ok && !bin_sort;
  uint32_t* bin_hist = nullptr;
  if (bin_ok) {
    ca.lo_rank = pb.lo_rank;
    ca.n_rank = pb.n_rank;
    ca.bin = sc.get<uint32_t>(g.R);
    bin_hist = sc.get<uint32_t>(nb);
    FIC_CUDA(cudaMemsetAsync(bin_hist, 0, nb * sizeof(uint32_t), s));
    ca.bin_hist = bin_hist;
  }
  k_classify<<<(unsigned)cdiv(g.R, 256), 256, 0, s>>>(ca);
  FIC_CHECK_LAUNCH();
  PlanCounts* d_pc = sc.get<PlanCounts>(1);
  if (bin_sort) {
    uint32_t* cursor = sc.get<uint32_t>(nb);
    k_bin_scan<<<1, 1024, 0, s>>>(bin_hist, nb, cursor, pb.n_rank + 1, g.R, d_pc);
    FIC_CHECK_LAUNCH();
    smem_optin_k(k_range_scatter, kMaxRangeBins * (int)sizeof(uint32_t));
    k_range_scatter<<<(unsigned)cdiv(g.R, 4096), 1024, nb * sizeof(uint32_t), s>>>(
        ca.bin, key, g.R, nb, cursor, key_s, rid_s);
    FIC_CHECK_LAUNCH();
  } else if (stable_sort) {
    // deterministic order (raster order inside a bin): every shard cuts the same list
    const int nchunk = (int)cdiv(g.R, kStableChunk);
    uint32_t* mat = sc.get<uint32_t>((size_t)nb * nchunk);
    uint32_t* start = sc.get<uint32_t>((size_t)nb * nchunk);
    smem_optin_k(k_chunk_hist, kMaxRangeBins * (int)sizeof(uint32_t));
    smem_optin_k(k_range_scatter_stable, kMaxRangeBins * (int)sizeof(uint32_t));
    k_chunk_hist<<<nchunk, 1024, nb * sizeof(uint32_t), s>>>(ca.bin, g.R, nb, nchunk, mat);
    FIC_CHECK_LAUNCH();
    k_bin_scan<<<1, 1024, 0, s>>>(mat, nb * nchunk, start, (pb.n_rank + 1) * nchunk, g.R, d_pc);
    FIC_CHECK_LAUNCH();
    k_range_scatter_stable<<<nchunk, 32, nb * sizeof(uint32_t), s>>>(ca.bin, key, g.R, nb, nchunk,
                                                                   start, key_s, rid_s);
    FIC_CHECK_LAUNCH();
  } else {
    // order by (class, lo) only (bits 32..63; stable, so ties keep raster order):
    // tiles need contiguous windows, and the result does not depend on the order
    cub_call(sc, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, key, key_s, rid, rid_s, g.R, 32, 64, s);
    });
  }
  if (!bin_sort) {
    unsigned long long* cum = sc.get<unsigned long long>(g.R);
    k_cost_scan<<<1, 1024, 0, s>>>(key_s, g.R, g.n_iso, cum);
    FIC_CHECK_LAUNCH();
    k_shard<<<1, 32, 0, s>>>(key_s, cum, g.R, shard, nshard, d_pc);
    FIC_CHECK_LAUNCH();
  }
  pmark();  // 10
  pmark();  // 11
  // Everything below is enqueued without waiting for the device: counts
  // live in PlanCounts / DevPlan, allocations use upper bounds.
  const int64_t n_tt_max = tensor_ok ? cdiv(g.R, RT) : 0;
  const int64_t n_er_max = g.R;
  int32_t* nslots = sc.get<int32_t>(g.R);
  FIC_CUDA(cudaMemsetAsync(nslots, 0, g.R * sizeof(int32_t), s));
  int32_t* wlo = sc.get<int32_t>(n_tt_max);
  int32_t* whi = sc.get<int32_t>(n_tt_max);
  int32_t* tnseg = sc.get<int32_t>(n_tt_max);
  int32_t* tbase = sc.get<int32_t>(n_tt_max);
  int32_t* enseg = sc.get<int32_t>(n_er_max);
  int32_t* ebase = sc.get<int32_t>(n_er_max);
  int64_t* sbase = sc.get<int64_t>(g.R);
  if (n_tt_max) {
    TileArgs ta{key_s, rid_s, d_pc, RT, seg_t, seg0, wlo, whi, tnseg, nslots, g.n_iso, counters + 3,
                nsub};
    k_tiles<<<(unsigned)cdiv(n_tt_max, 128), 128, 0, s>>>(ta);
    FIC_CHECK_LAUNCH();
  }
  k_exact_segs<<<(unsigned)cdiv(n_er_max, 256), 256, 0, s>>>(key_s, rid_s, d_pc, seg_e, enseg, nslots);
  FIC_CHECK_LAUNCH();
  constexpr int kSplitCap = 2 * 148;  // tail items run as pieces (TcArgs::n_split)
  DevPlan* d_plan = &d_rb->plan;
  k_plan_scans<<<3, 1024, 0, s>>>(tnseg, tbase, enseg, ebase, nslots, sbase, g.R, d_pc, RT, nsub,
                                  kSplitCap, d_plan);
  FIC_CHECK_LAUNCH();
  pmark();  // 12
  // upper bounds of the item / slot counts (a shard or class can only be smaller)
  const int64_t segs_max = 1 + cdiv(std::max<int64_t>(g.D - seg0, 0), seg_t);
  const int64_t esegs_max = tensor_ok ? std::max<int64_t>(1, cdiv(std::min<int64_t>(small_pool - 1, g.D), seg_e))
                                      : cdiv(g.D, seg_e);
  int64_t titems_n = n_tt_max * segs_max, eitems_n = n_er_max * esegs_max;
  int64_t slots_n = (int64_t)g.R * std::max<int64_t>(segs_max * nsub, esegs_max);
  const double bound_bytes = 8.0 * (titems_n + eitems_n) + (double)sizeof(Partial) * slots_n;
  if (bound_bytes > (double)(1ll << 30) || getenv("FIC_PLAN_SYNC")) {
    // bounds too loose (e.g. the exact matcher on a large image): read the counts
    DevPlan hp;
    FIC_CUDA(cudaMemcpyAsync(&hp, d_plan, sizeof(hp), cudaMemcpyDeviceToHost, s));
    FIC_CUDA(cudaStreamSynchronize(s));
    titems_n = hp.n_titems;
    eitems_n = hp.n_eitems;
    slots_n = hp.n_slots;
  }
  pmark();  // 13
  int2* titems = sc.get<int2>(titems_n);
  int2* eitems = sc.get<int2>(eitems_n);
  Partial* partials = sc.get<Partial>(slots_n);
  if (n_tt_max) {
    // segment-major order: every tile's first segment runs before any second
    // segment, so later segments start from the thresholds the earlier ones found
    const int smax = (int)segs_max;
    uint32_t* shist = sc.get<uint32_t>(smax + 1);
    uint32_t* sbase2 = sc.get<uint32_t>(smax);
    uint32_t* scur = sc.get<uint32_t>(smax);
    FIC_CUDA(cudaMemsetAsync(shist, 0, (smax + 1) * sizeof(uint32_t), s));
    k_seg_hist<<<(unsigned)cdiv(n_tt_max, 256), 256, 0, s>>>(tnseg, d_plan, smax, shist);
    FIC_CHECK_LAUNCH();
    k_seg_base<<<1, 32, 0, s>>>(shist, smax, sbase2, scur);
    FIC_CHECK_LAUNCH();
    k_seg_place<<<(unsigned)smax, 1024, 0, s>>>(tnseg, d_plan, sbase2, titems);
    FIC_CHECK_LAUNCH();
  }
  k_expand<<<(unsigned)cdiv(n_er_max, 128), 128, 0, s>>>(enseg, ebase, d_plan, eitems);
  FIC_CHECK_LAUNCH();

  pmark();  // 14
  FIC_CUDA(cudaStreamWaitEvent(s, side.ev[2], 0));  // join: pool + ranges
  PoolView P = pool_view(pa);
  RangeView Rv{ra.info, ra.rows, pb.lo, pb.hi, g.n_iso, K, ra.KP};
  tm.mark();  // 3
  SlArgs sla{};                    // survivor list (k_sl_rescore)
  HlArgs hla{};                    // hit list (k_hl_rescore)
  // FIC_PRIME_THR (experiment only): the tensor matcher's per-range
  // thresholds start from the final errors of the previous call with the
  // same R on this device -- how much of K4 is threshold discovery
  static std::map<std::pair<int, int>, unsigned long long*> prime_cache;
  static std::mutex prime_mu;
  unsigned long long* prime_buf = nullptr;
  bool prime_ok = false;
  if (getenv("FIC_PRIME_THR")) {
    std::lock_guard<std::mutex> lock(prime_mu);
    auto& pb2 = prime_cache[{dev_id, g.R}];
    prime_ok = pb2 != nullptr;
    if (!pb2) FIC_CUDA(cudaMalloc(&pb2, g.R * 8));
    prime_buf = pb2;
  }
  if (n_tt_max && titems_n) {
    unsigned long long* thr_g = sc.get<unsigned long long>(g.R);
    k_fill_u64<<<(unsigned)cdiv(g.R, 256), 256, 0, s>>>(thr_g, 0x7ff0000000000000ull, g.R);
    if (prime_buf && prime_ok)  // experiment: start from the previous call's final errors
      FIC_CUDA(cudaMemcpyAsync(thr_g, prime_buf, g.R * 8, cudaMemcpyDeviceToDevice, s));
    FIC_CHECK_LAUNCH();
    constexpr int BN_COLS = 128;
    TcArgs ta{titems, titems_n, rid_s, n_tt_max * RT, wlo, whi, seg_t, seg0, RT, sbase, partials,
              counters, counters + 15, thr_g, 0, nullptr};
    ta.nsub = nsub;
    // A pilot item per tile seeds the thresholds before the main items.
    // 4x4 ranges (K = 16): the fp16 screen keeps ~0.1% of the candidates and
    // thresholds found along the way arrive too late, so the pilot samples
    // every 8th N-tile of each window and every survivor goes to the lists
    // (cfg4: 142 -> 33 ms).  8x8 ranges sample about
    // pilot_samples N-tiles of each window (adaptive stride; cfg3 -0.08 ms)
    // and keep the rescoring warp.
    const bool k16 = K == 16;
    ta.pilot_cols = getenv("FIC_PILOT") ? std::max(0, atoi(getenv("FIC_PILOT"))) / BN_COLS * BN_COLS
                                        : (tc_tile_rows(K) == 128 ? (1 << 30) : 0);  // (not the CTA-pair variant)
    ta.pilot_stride = getenv("FIC_PILOT_STRIDE") ? std::max(0, atoi(getenv("FIC_PILOT_STRIDE")))
                                                 : (k16 ? 8 : 0);
    ta.pilot_samples = getenv("FIC_PILOT_SAMPLES") ? std::max(1, atoi(getenv("FIC_PILOT_SAMPLES"))) : 16;
    ta.n_split = nsub > 1 ? std::min<int64_t>(titems_n, kSplitCap) : 0;  // bound
    ta.plan = d_plan;
    if (flat_path) {
      ta.flat_c = fl.flat_c;
      ta.flat_canon = fl.canon;
    }
    if (getenv("FIC_SL") ? atoi(getenv("FIC_SL")) != 0 : k16) {
      // survivor list (TcArgs::sl; default for 4x4 ranges with the pilot,
      // without good starting thresholds the list grows to billions of
      // candidates at cfg4): 16-byte entries, capacity
      // min(128 M, max(1 M, 2048 R)) (2 GB at most)
      ta.sl_cap = (uint32_t)std::min<int64_t>(128 << 20, std::max<int64_t>(1 << 20, 2048 * (int64_t)g.R));
      if (getenv("FIC_SL_CAP")) ta.sl_cap = (uint32_t)std::max(1, atoi(getenv("FIC_SL_CAP")));
      ta.sl = sc.get<uint4>(ta.sl_cap);
      ta.sl_count = d_rb->sl_count;
      ta.sl_all = getenv("FIC_SL_ALL") ? atoi(getenv("FIC_SL_ALL")) : (k16 ? 1 : 0);
      sla.sl = ta.sl;
      sla.sl_count = ta.sl_count;
      sla.sl_cap = ta.sl_cap;
      sla.best = sc.get<unsigned long long>(2 * (size_t)g.R);
      sla.pre = sc.get<unsigned long long>(g.R);
      sla.counters = counters;
      k_sl_init<<<(unsigned)cdiv(g.R, 256), 256, 0, s>>>(sla.best, sla.pre, g.R);
      FIC_CHECK_LAUNCH();
      // hit list (every survivor to the lists): one entry per hit warp-chunk,
      // capacity min(128 M, max(1 M, 512 R)) entries; FIC_HL=0 turns it off
      if (ta.sl_all == 1 && (!getenv("FIC_HL") || atoi(getenv("FIC_HL")) != 0)) {
        ta.hl_cap = (uint32_t)std::min<int64_t>(128 << 20, std::max<int64_t>(1 << 20, 512 * (int64_t)g.R));
        if (getenv("FIC_HL_CAP")) ta.hl_cap = (uint32_t)std::max(1, atoi(getenv("FIC_HL_CAP")));
        ta.hl = sc.get<uint4>(ta.hl_cap);
        ta.hl_count = d_rb->sl_count + 1;
        hla.hl = ta.hl;
        hla.hl_count = ta.hl_count;
        hla.hl_cap = ta.hl_cap;
        hla.tlist = rid_s;
        hla.plan = d_plan;
        hla.thr_g = thr_g;
        hla.best = sla.best;
        hla.pre = sla.pre;
        hla.counters = counters;
        hla.tests = &d_rb->hl_tests;
        if (!getenv("FIC_HL_SORT") || atoi(getenv("FIC_HL_SORT")) != 0) {
          hla.sorted = sc.get<uint4>(ta.hl_cap);
          hla.n_sorted = d_rb->sl_count + 2;
          hla.run_ctr = d_rb->sl_count + 3;  // zeroed with the readback block
          hla.bins = sc.get<uint32_t>((size_t)(g.D + 63) / 64 + 2);
        }
      }
    }
    const char* dbg_env = getenv("FIC_TC_DEBUG");
    if (dbg_env && (atoi(dbg_env) & (32 | 8192))) {
      ta.dbg = sc.get<unsigned long long>(64 * 24);
      FIC_CUDA(cudaMemsetAsync(ta.dbg, 0, 64 * 24 * 8, s));
    }
    launch_tc(P, Rv, ta, s);
    if (ta.dbg && (atoi(dbg_env) & 8192)) {  // per-CTA start / end: the tail of the persistent grid
      std::vector<unsigned long long> h(64 * 24);
      FIC_CUDA(cudaMemcpyAsync(h.data(), ta.dbg, h.size() * 8, cudaMemcpyDeviceToHost, s));
      FIC_CUDA(cudaStreamSynchronize(s));
      int n = 0;
      unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
      double em = 0, im = 0;
      unsigned long long imin = ~0ull, imax = 0;
      for (int b = 0; b < 512 && h[2 * b + 1]; ++b, ++n) {
        s0 = std::min(s0, h[2 * b]);
        s1 = std::max(s1, h[2 * b]);
        e0 = std::min(e0, h[2 * b + 1]);
        e1 = std::max(e1, h[2 * b + 1]);
        em += (double)h[2 * b + 1];
        im += (double)h[1024 + b];
        imin = std::min(imin, h[1024 + b]);
        imax = std::max(imax, h[1024 + b]);
      }
      if (n)
        fprintf(stderr, "tc tail: %d CTAs, start spread %.1f us, end min %.1f mean %.1f max %.1f us after first start; items/CTA %llu..%llu mean %.1f\n",
                n, (s1 - s0) / 1e3, (e0 - s0) / 1e3, (em / n - (double)s0) / 1e3, (e1 - s0) / 1e3, imin, imax, im / n);
    } else if (ta.dbg) {
      std::vector<unsigned long long> h(64 * 24);
      FIC_CUDA(cudaMemcpyAsync(h.data(), ta.dbg, h.size() * 8, cudaMemcpyDeviceToHost, s));
      FIC_CUDA(cudaStreamSynchronize(s));
      unsigned long long t0 = h[0];
      fprintf(stderr, "tile: tma_issue mma_issue mma_tempty_ok | screener (group j%%2, quarter 0): tfull_ok ld0_done ld1_done\n");
      for (int j = 0; j < 64; ++j) {
        fprintf(stderr, "%3d: %7lld %7lld %7lld |", j, (long long)(h[j * 24] - t0), (long long)(h[j * 24 + 1] - t0),
                (long long)(h[j * 24 + 2] - t0));
        for (int w = 4; w < 7; ++w) fprintf(stderr, " %7lld", (long long)(h[j * 24 + w] - t0));
        fprintf(stderr, "\n");
      }
    }
  }
  FIC_CUDA(record_timing_event(tm.ev[21], s));
  launch_sl_rescore(P, Rv, sla, s);
  launch_hl_sort(hla, g.D, s);
  launch_hl_rescore(P, Rv, hla, s);
  FIC_CUDA(record_timing_event(tm.ev[22], s));
  tm.mark();  // 4
  if (eitems_n) {
    ExactArgs ea{eitems, eitems_n, rid_s, seg_e, sbase, partials, counters, d_plan};
    launch_exact(P, Rv, ea, s);
  }
  tm.mark();  // 5
  MergeArgs ma{g.R, sbase, nslots, partials, records, pre_rms, post_rms, (double)K, sla.best,
               sla.pre, prime_buf};
  launch_merge(ma, s);
  tm.mark();  // 6
  FIC_CUDA(cudaMemcpyAsync(h_rb, d_rb, sizeof(Readback), cudaMemcpyDeviceToHost, s));
  tm.mark();  // 7
  post.flat_path = flat_path;
  post.fl = fl;
  post.P = P;
  post.lo = pb.lo;
  post.hi = pb.hi;
  post.nslots = nslots;
  post.sl_cap = sla.sl_cap;
  post.hl_cap = hla.hl_cap;
  post.launches = g_launches;
  post.sc_off = sc.offset();
  return post;
  };

  EncPost post;
  int graph_mode = 0;  // fic_stats_t::graph
  GraphKey gk;
  const bool elig = !g_graphs_off && st != nullptr && (int64_t)H * W <= (int64_t)4096 * 4096 &&
                    graphs_allowed();
  if (elig) {
    gk.v = {dev_id, (int64_t)(uintptr_t)s, (int64_t)(uintptr_t)img, H, W,
            (int64_t)(uintptr_t)records, (int64_t)(uintptr_t)pre_rms, (int64_t)(uintptr_t)post_rms,
            (int64_t)(uintptr_t)pool_sizes, (int64_t)(uintptr_t)sc.arena_base(), (int64_t)sc.arena_cap(),
            p.range_size, p.domain_size, p.stride, p.isometries, p.strategy, p.fd_source, p.has_delta,
            p.matcher, (int64_t)(uintptr_t)p.h_ln_table, p.ln_len, p.shard_index, p.shard_count,
            p.max_segment, p.small_pool, p.n_fd_weights_dom, p.n_fd_weights_rng};
    int64_t bits;
    std::memcpy(&bits, &p.delta, 8);
    gk.v.push_back(bits);
    for (int i = 0; i < p.n_fd_weights_dom && p.h_fd_weights_dom; ++i) {
      std::memcpy(&bits, p.h_fd_weights_dom + i, 8);
      gk.v.push_back(bits);
    }
    for (int i = 0; i < p.n_fd_weights_rng && p.h_fd_weights_rng; ++i) {
      std::memcpy(&bits, p.h_fd_weights_rng + i, 8);
      gk.v.push_back(bits);
    }
  }
  auto hit = elig ? g_graphs.find(gk) : g_graphs.end();
  // the graph stream, ordered after the caller's stream (and back, below)
  auto to_graph_stream = [&]() -> GraphStream& {
    GraphStream& G = GraphStream::get(dev_id);
    FIC_CUDA(cudaEventRecord(G.in, s_user));
    FIC_CUDA(cudaStreamWaitEvent(G.gs, G.in, 0));
    s = G.gs;
    return G;
  };
  auto back_to_user_stream = [&](GraphStream& G) {
    FIC_CUDA(cudaEventRecord(G.out, G.gs));
    s = s_user;
    FIC_CUDA(cudaStreamWaitEvent(s_user, G.out, 0));
  };
  if (hit != g_graphs.end()) {  // replay
    post = hit->second.post;
    sc.restore(post.sc_off);
    GraphStream& G = to_graph_stream();
    FIC_CUDA(cudaGraphLaunch(hit->second.exec, G.gs));
    back_to_user_stream(G);
    graph_mode = 2;
  } else if (elig && g_graph_seen.count(gk) && sc.fits()) {  // record, then launch
    const size_t off0 = sc.offset();
    const int l0 = g_launches;
    bool ok = true;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    GraphStream& G = to_graph_stream();
    FIC_CUDA(cudaStreamBeginCapture(G.gs, cudaStreamCaptureModeThreadLocal));
    g_capturing = true;
    try {
      post = enqueue();
    } catch (...) {
      ok = false;
    }
    g_capturing = false;
    if (cudaStreamEndCapture(G.gs, &graph) != cudaSuccess || !graph) ok = false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(G.gs, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone ||
        cudaStreamIsCapturing(side.s2, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      g_graphs_off = true;  // should not happen; never capture again in this thread
    if (ok && sc.spilled()) ok = false;  // an allocation outside the arena: not replayable
    if (ok && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) ok = false;
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (ok) {
      if (g_graphs.size() >= 16) {
        for (auto& kv : g_graphs) cudaGraphExecDestroy(kv.second.exec);
        g_graphs.clear();
      }
      g_graphs[gk] = GraphEnt{exec, post};
      FIC_CUDA(cudaGraphLaunch(exec, G.gs));
      back_to_user_stream(G);
      graph_mode = 1;
    } else {  // the direct path on the caller's stream
      if (exec) cudaGraphExecDestroy(exec);
      s = s_user;
      sc.restore(off0);
      g_launches = l0;
      post = enqueue();
    }
  } else {
    if (elig) {
      if (g_graph_seen.size() > 256) g_graph_seen.clear();
      g_graph_seen.insert(gk);
    }
    post = enqueue();
  }
  g_launches = post.launches;
  FIC_CUDA(cudaStreamSynchronize(s));
  const Readback& hrb = *h_rb;
  const bool flat_path = post.flat_path;
  FlatArgs fl = post.fl;
  const PoolView P = post.P;
  int32_t* nslots = post.nslots;
  const unsigned long long* hc = hrb.counters;
  const double* hs = hrb.scal;
  const DevPlan& hp = hrb.plan;
  const unsigned long long n_flat = flat_path ? hrb.flat[0] : 0;
  if (n_flat) {  // flat ranges on the canonical slab: one reduction per pixel value
    fl.lo = post.lo;
    fl.hi = post.hi;
    fl.nslots = nslots;
    fl.present = sc.get<uint8_t>(256);
    fl.nchunk = (int)cdiv(g.D, 4096);
    fl.part = sc.get<FlatArgs::Best>((size_t)256 * fl.nchunk);
    fl.best = sc.get<FlatArgs::Best>(256);
    fl.records = records;
    fl.pre_rms = pre_rms;
    fl.post_rms = post_rms;
    launch_flat_match(P, fl, s);
    FIC_CUDA(cudaEventRecord(tm.ev[23], s));  // end of the flat fix-up (event 23: not a plan mark)
    FIC_CUDA(cudaStreamSynchronize(s));
  }
  sc.verify("encode");
  if (ptime && pn == 15) {
    fprintf(stderr, "plan timing (ms): fd %.3f pool(side) %.3f | fork %.3f - %.3f classify..shard %.3f sync1 %.3f "
            "tiles..totals %.3f sync2 %.3f items %.3f | tensor %.3f exact %.3f merge %.3f readback %.3f | seed rounds %llu hit rounds %llu hit lanes %llu\n",
            tm.ms(0, 1), [&] { float t = 0; cudaEventElapsedTime(&t, side.ev[3], side.ev[4]); return (double)t; }(), tm.ms(2, 8), tm.ms(8, 9), tm.ms(9, 10), tm.ms(10, 11), tm.ms(11, 12),
            tm.ms(12, 13), tm.ms(13, 14), tm.ms(3, 4), tm.ms(4, 5), tm.ms(5, 6), tm.ms(6, 7), hc[14], hc[12], hc[13]);
  }
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->n_ranges = g.R;
    st->n_domains = g.D;
    st->comparisons = (int64_t)hc[2] * g.n_iso;
    st->mean_pool_size = (double)hc[2] / (double)g.R;
    st->fd_min = hs[0];
    st->fd_max = hs[1];
    st->half_width = p.strategy == FIC_DYNAMIC_FD ? hs[2] : 0.0;
    st->ms_fd = tm.ms(0, 1);
    {
      float t = 0;
      cudaEventElapsedTime(&t, side.ev[3], side.ev[4]);
      st->ms_pool = t;
      t = 0;
      cudaEventElapsedTime(&t, side.ev[5], side.ev[4]);
      st->ms_pool_main = t;
    }
    st->ms_match = tm.ms(3, 6);
    st->ms_tensor = tm.ms(3, 21);
    st->ms_sl = tm.ms(21, 22);
    st->sl_entries = std::min<int64_t>(hrb.sl_count[0], post.sl_cap);
    st->hl_entries = std::min<int64_t>(hrb.sl_count[1], post.hl_cap);
    st->hl_tests = (int64_t)hrb.hl_tests;
    st->ms_exact = tm.ms(4, 5);
    st->ms_total = n_flat ? tm.ms(0, 23) : tm.ms(0, 7);
    st->exact_evals = (int64_t)hc[0];
    st->tensor_candidates = (int64_t)hc[1];
    st->tensor_comparisons = (int64_t)hc[3];
    st->tensor_tiles = (int32_t)hp.n_tt;
    st->exact_tiles = (int32_t)hp.n_er;
    st->work_items = (int32_t)(hp.n_titems + hp.n_eitems);
    st->kernel_launches = g_launches;
    st->graph = graph_mode;
    if ((getenv("FIC_TC_DEBUG") && (atoi(getenv("FIC_TC_DEBUG")) & 4)) || getenv("FIC_TC_PROF"))
      fprintf(stderr, "tc cycles: producer-empty %.3g  mma-tempty %.3g  mma-full %.3g  epi-tfull %.3g  epi-slow %.3g  epi-total %.3g  mma-loop %.3g  setup %.3g  teardown(tma warp) %.3g  items %.0f\n",
              (double)hc[4], (double)hc[5], (double)hc[6], (double)hc[7], (double)hc[8], (double)hc[9], (double)hc[10], (double)hc[11], (double)hc[12], (double)hc[13]);
  }
}

// K1 outputs in pool order, for the parity tests (fic_pool_v1): the
// decimated pixels come through the same DomSrc gather the matchers use.
template <int K>
__global__ void k_dom_gather(PoolView P, uint8_t* dec) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P.D) return;
  uint32_t w[K / 4];
  dom_words<K>(P, p, pool_id(P, p), w);
  uint32_t* o = reinterpret_cast<uint32_t*>(dec + (size_t)p * K);
#pragma unroll
  for (int i = 0; i < K / 4; ++i) o[i] = w[i];
}

__global__ void k_raw_gather(PoolView P, int K, uint8_t* dec) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P.D) return;
  for (int k = 0; k < K; ++k) dec[(size_t)p * K + k] = P.src.raw[(size_t)p * P.src.KP + k];
}

static void pool_impl(const uint8_t* img, int H, int W, const fic_params_t& p, int64_t* order,
                      uint8_t* dec, uint32_t* sums, double* inv_den, uint16_t* b_rows,
                      cudaStream_t s) {
  Geo g = validate(H, W, p);
  if (p.strategy == FIC_STATIC2 || p.strategy == FIC_DYNAMIC_FD) {
    check_dbc_side(p.fd_source == FIC_FD_ORIGINAL ? g.ds : g.rs);
    check_dbc_side(g.rs);
  }
  const int K = g.npx;
  const bool tensor_ok = tc_supported(K);
  if (b_rows && !tensor_ok) invalid("fp16 B rows exist for 4x4 and 8x8 ranges only");
  Scratch sc(s);
  PlanBufs pb = make_plan(sc, s, img, g, p, false, true);
  PoolArgs pa = pool_args(sc, g, img, pb.order, tensor_ok);
  launch_pool(pa, s);
  const PoolView P = pool_view(pa);
  const unsigned blocks = (unsigned)cdiv(g.D, 256);
  if (order) {
    if (pb.order) {
      k_u32_to_i64<<<blocks, 256, 0, s>>>(pb.order, order, g.D);
    } else {
      uint32_t* io = sc.get<uint32_t>(g.D);
      k_iota<<<blocks, 256, 0, s>>>(io, g.D);
      k_u32_to_i64<<<blocks, 256, 0, s>>>(io, order, g.D);
    }
    FIC_CHECK_LAUNCH();
  }
  if (dec) {
    if (K == 64)
      k_dom_gather<64><<<blocks, 256, 0, s>>>(P, dec);
    else if (K == 16)
      k_dom_gather<16><<<blocks, 256, 0, s>>>(P, dec);
    else
      k_raw_gather<<<blocks, 256, 0, s>>>(P, K, dec);
    FIC_CHECK_LAUNCH();
  }
  if (sums)
    FIC_CUDA(cudaMemcpyAsync(sums, pa.sums, g.D * sizeof(uint2), cudaMemcpyDeviceToDevice, s));
  if (inv_den)
    FIC_CUDA(cudaMemcpyAsync(inv_den, pa.inv_den, g.D * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (b_rows)
    FIC_CUDA(cudaMemcpyAsync(b_rows, pa.bh, (size_t)g.D * K * 2, cudaMemcpyDeviceToDevice, s));
  FIC_CUDA(cudaStreamSynchronize(s));
  sc.verify("pool");
}

static void plan_impl(const uint8_t* img, int H, int W, const fic_params_t& p, double* fd_dom,
                      double* fd_rng, int64_t* order, int64_t* slab_lo, int64_t* slab_hi,
                      fic_stats_t* st, cudaStream_t s) {
  Geo g = validate(H, W, p);
  if (p.strategy == FIC_STATIC2 || p.strategy == FIC_DYNAMIC_FD) {
    check_dbc_side(p.fd_source == FIC_FD_ORIGINAL ? g.ds : g.rs);
    check_dbc_side(g.rs);
  }
  Scratch sc(s);
  PlanBufs pb = make_plan(sc, s, img, g, p, fd_dom != nullptr, true);
  if (fd_dom && pb.fd_dom)
    FIC_CUDA(cudaMemcpyAsync(fd_dom, pb.fd_dom, g.D * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (fd_rng && pb.fd_rng)
    FIC_CUDA(cudaMemcpyAsync(fd_rng, pb.fd_rng, g.R * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (order) {
    if (pb.order) {
      k_u32_to_i64<<<(unsigned)cdiv(g.D, 256), 256, 0, s>>>(pb.order, order, g.D);
    } else {
      uint32_t* io = sc.get<uint32_t>(g.D);
      k_iota<<<(unsigned)cdiv(g.D, 256), 256, 0, s>>>(io, g.D);
      k_u32_to_i64<<<(unsigned)cdiv(g.D, 256), 256, 0, s>>>(io, order, g.D);
    }
    FIC_CHECK_LAUNCH();
  }
  if (slab_lo) k_i32_to_i64<<<(unsigned)cdiv(g.R, 256), 256, 0, s>>>(pb.lo, slab_lo, g.R);
  if (slab_hi) k_i32_to_i64<<<(unsigned)cdiv(g.R, 256), 256, 0, s>>>(pb.hi, slab_hi, g.R);
  FIC_CHECK_LAUNCH();
  double hs[4];
  FIC_CUDA(cudaMemcpyAsync(hs, pb.scal, sizeof(hs), cudaMemcpyDeviceToHost, s));
  FIC_CUDA(cudaStreamSynchronize(s));
  sc.verify("plan");
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->n_ranges = g.R;
    st->n_domains = g.D;
    st->fd_min = hs[0];
    st->fd_max = hs[1];
    st->half_width = p.strategy == FIC_DYNAMIC_FD ? hs[2] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// decode (codec.py:534-598): gather 2x2 means, isometry, s*x + o, clip,
// scatter; the work image stays float64, rint -> uint8 when yielded.
// ---------------------------------------------------------------------------
struct DecArgs {
  const uint8_t* rec;
  int W, rs, st, ndx, nrx, R;
  uint32_t n_dom;
  const int* perm;  // [8][K]
  const double* src;
  double* dst;
  uint8_t* out;     // optional: rint(dst) as uint8 (one decode_iterates snapshot)
};

__global__ void k_decode(DecArgs a) {
  int K = a.rs * a.rs;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)a.R * K) return;
  int r = (int)(t / K), k = (int)(t - (int64_t)r * K);
  const uint8_t* rc = a.rec + (int64_t)r * 7;
  uint32_t dom = rc[0] | (rc[1] << 8) | (rc[2] << 16) | ((uint32_t)rc[3] << 24);
  if (dom >= a.n_dom) dom = 0;  // memory safety only: callers validate first
  int iso = rc[4];
  double s_hat = __dsub_rn(__dmul_rn((double)rc[5], 2.0 / 31.0), 1.0);
  double o_hat = __dsub_rn(__dmul_rn((double)rc[6], 510.0 / 127.0), 255.0);
  // domains[rows][:, perms[iso]] for iso 0..7; other bytes keep the identity
  // (codec.py:580-592 permutes only the rows of isometries 0..7)
  int m = iso < 8 ? a.perm[iso * K + k] : k;
  int u = m / a.rs, v = m - u * a.rs;
  int64_t y = (int64_t)(dom / a.ndx) * a.st + 2 * u;
  int64_t x = (int64_t)(dom % a.ndx) * a.st + 2 * v;
  int64_t gi = y * a.W + x;
  double sum = __dadd_rn(__dadd_rn(__dadd_rn(a.src[gi], a.src[gi + 1]), a.src[gi + a.W]),
                         a.src[gi + a.W + 1]);
  double d = __dmul_rn(0.25, sum);
  double val = __dadd_rn(__dmul_rn(s_hat, d), o_hat);
  val = fmin(fmax(val, 0.0), 255.0);
  int ry = r / a.nrx, rx = r - ry * a.nrx;
  int64_t oy = (int64_t)ry * a.rs + k / a.rs, ox = (int64_t)rx * a.rs + k % a.rs;
  a.dst[oy * a.W + ox] = val;
  if (a.out) a.out[oy * a.W + ox] = (uint8_t)rint(val);
}

__global__ void k_fill(double* w, int64_t n, double v, const uint8_t* init) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = init ? (double)init[i] : v;
}

__global__ void k_max_domain(const uint8_t* rec, int R, unsigned int* mx) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const uint8_t* rc = rec + (int64_t)r * 7;
  atomicMax(mx, rc[0] | (rc[1] << 8) | (rc[2] << 16) | ((uint32_t)rc[3] << 24));
}

// Validation of decode_iterates (codec.py:541-556), reference texts.
static DecArgs decode_geometry(const uint8_t* rec, int H, int W, int rs, int ds, int st,
                               int iters) {
  if (iters < 1) invalid("iterations must be >= 1");
  if (rs <= 0 || H % rs || W % rs)
    invalid("image " + std::to_string(W) + "x" + std::to_string(H) +
            " not divisible by range size " + std::to_string(rs));
  if (st < 1) invalid("stride must be >= 1");
  if (ds > std::min(W, H))
    invalid("domain size " + std::to_string(ds) + " exceeds image " + std::to_string(W) + "x" +
            std::to_string(H));
  DecArgs a{};
  a.rec = rec;
  a.W = W;
  a.rs = rs;
  a.st = st;
  a.ndx = (W - ds) / st + 1;
  a.nrx = W / rs;
  a.R = (W / rs) * (H / rs);
  const int ndy = (H - ds) / st + 1;
  a.n_dom = (uint32_t)((int64_t)a.ndx * ndy);
  // the 2x2 gathers of the last domain must stay inside the image (numpy
  // raises IndexError there, codec.py:575-582)
  if ((int64_t)(a.ndx - 1) * st + 2 * rs > W || (int64_t)(ndy - 1) * st + 2 * rs > H)
    invalid("index out of bounds: domain_size too small for range_size in this geometry");
  return a;
}

// isometry permutation tables on the device, once per (device, range size)
static const int* iso_perm_table(int rs) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, int*> cache;
  int dev = 0;
  FIC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, rs});
  if (it != cache.end()) return it->second;
  const int K = rs * rs;
  std::vector<int> perm(8 * K), inv(8 * K);
  iso_tables(rs, perm.data(), inv.data());
  int* d = nullptr;
  FIC_CUDA(cudaMalloc(&d, 8 * K * sizeof(int)));
  FIC_CUDA(cudaMemcpy(d, perm.data(), 8 * K * sizeof(int), cudaMemcpyHostToDevice));
  cache.emplace(std::make_pair(dev, rs), d);
  return d;
}

static void decode_impl(const uint8_t* rec, int H, int W, int rs, int ds, int st, int iters,
                        double initial, const uint8_t* init_img, uint8_t* out, cudaStream_t s) {
  DecArgs a = decode_geometry(rec, H, W, rs, ds, st, iters);
  Scratch sc(s);
  // records referencing a domain outside the geometry (codec.py:551-555)
  unsigned int* d_mx = sc.get<unsigned int>(1);
  FIC_CUDA(cudaMemsetAsync(d_mx, 0, sizeof(unsigned int), s));
  k_max_domain<<<(unsigned)cdiv(a.R, 256), 256, 0, s>>>(rec, a.R, d_mx);
  FIC_CHECK_LAUNCH();
  unsigned int mx = 0;
  FIC_CUDA(cudaMemcpyAsync(&mx, d_mx, sizeof(mx), cudaMemcpyDeviceToHost, s));
  FIC_CUDA(cudaStreamSynchronize(s));
  if (a.R && mx >= a.n_dom) invalid("record references a domain outside the current image geometry");
  a.perm = iso_perm_table(rs);
  int64_t n = (int64_t)H * W;
  double* w0 = sc.get<double>(n);
  double* w1 = sc.get<double>(n);
  k_fill<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(w0, n, initial, init_img);
  FIC_CHECK_LAUNCH();
  for (int i = 0; i < iters; ++i) {
    a.src = w0;
    a.dst = w1;
    a.out = (i == iters - 1) ? out : nullptr;
    k_decode<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(a);
    FIC_CHECK_LAUNCH();
    std::swap(w0, w1);
  }
  FIC_CUDA(cudaStreamSynchronize(s));
  sc.verify("decode");
}

static void decode_step_impl(const uint8_t* rec, int H, int W, int rs, int ds, int st,
                             const double* src, double* dst, uint8_t* out, cudaStream_t s) {
  DecArgs a = decode_geometry(rec, H, W, rs, ds, st, 1);
  if (!src || !dst) invalid("work images must not be NULL");
  a.perm = iso_perm_table(rs);
  a.src = src;
  a.dst = dst;
  a.out = out;
  const int64_t n = (int64_t)H * W;
  k_decode<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
}

}  // namespace fic

// ===========================================================================
// Multi-GPU exchange of range sharding (sharding.py): each rank's outputs
// packed into an int64 (R, 3) buffer -- record bytes plus an owner-count
// byte, pre and post RMS bits -- zero outside the ranges the rank matched
// (post RMS >= 0), so one all-reduce (SUM) over the ranks reproduces every
// range's bytes; the unpack writes them back and counts ranges whose owner
// count is not 1 (a hole or an overlap in the partition).
__global__ void k_shard_pack(const uint8_t* rec, const double* pre, const double* post, int64_t n,
                             unsigned long long* buf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double p = post[i];
  unsigned long long w0 = 0, w1 = 0, w2 = 0;
  if (p >= 0.0) {
    const uint8_t* r = rec + i * 7;
    for (int k = 0; k < 7; ++k) w0 |= (unsigned long long)r[k] << (8 * k);
    w0 |= 1ull << 56;
    w1 = (unsigned long long)__double_as_longlong(pre[i]);
    w2 = (unsigned long long)__double_as_longlong(p);
  }
  buf[3 * i] = w0;
  buf[3 * i + 1] = w1;
  buf[3 * i + 2] = w2;
}

__global__ void k_shard_unpack(const unsigned long long* buf, int64_t n, uint8_t* rec, double* pre,
                               double* post, unsigned int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = i < n && (buf[3 * i] >> 56) == 1;
  if (i < n) {
    const unsigned long long w0 = buf[3 * i];
    for (int k = 0; k < 7; ++k) rec[i * 7 + k] = (uint8_t)(w0 >> (8 * k));
    pre[i] = __longlong_as_double((long long)buf[3 * i + 1]);
    post[i] = __longlong_as_double((long long)buf[3 * i + 2]);
  }
  const unsigned m = __ballot_sync(0xffffffffu, i < n && !ok);
  if (m && (threadIdx.x & 31) == 0) atomicAdd(bad, (unsigned)__popc(m));
}

// extern "C"
// ===========================================================================
using namespace fic;

extern "C" int fic_encode_v1(const uint8_t* d_image, int32_t height, int32_t width,
                             const fic_params_t* params, uint8_t* d_records, double* d_pre_rms,
                             double* d_post_rms, int64_t* d_pool_sizes, fic_stats_t* h_stats,
                             void* stream) {
  return guarded([&] {
    if (!params) invalid("params must not be NULL");
    encode_impl(d_image, height, width, *params, d_records, d_pre_rms, d_post_rms, d_pool_sizes,
                h_stats, as_stream(stream));
  });
}

extern "C" int fic_plan_v1(const uint8_t* d_image, int32_t height, int32_t width,
                           const fic_params_t* params, double* d_fd_dom, double* d_fd_rng,
                           int64_t* d_order, int64_t* d_slab_lo, int64_t* d_slab_hi,
                           fic_stats_t* h_stats, void* stream) {
  return guarded([&] {
    if (!params) invalid("params must not be NULL");
    plan_impl(d_image, height, width, *params, d_fd_dom, d_fd_rng, d_order, d_slab_lo, d_slab_hi,
              h_stats, as_stream(stream));
  });
}

extern "C" int fic_pool_v1(const uint8_t* d_image, int32_t height, int32_t width,
                           const fic_params_t* params, int64_t* d_order, uint8_t* d_decimated,
                           uint32_t* d_sums, double* d_inv_den, uint16_t* d_b_rows,
                           void* stream) {
  return guarded([&] {
    if (!params) invalid("params must not be NULL");
    pool_impl(d_image, height, width, *params, d_order, d_decimated, d_sums, d_inv_den, d_b_rows,
              as_stream(stream));
  });
}

extern "C" int fic_dbc_v2(const uint8_t* d_blocks, int64_t n, int32_t side, int32_t gray_levels, int32_t clamp,
                          const double* h_ln_table, int32_t ln_len, const double* h_weights,
                          int32_t n_weights, double* d_fd, void* stream) {
  return guarded([&] {
    if (gray_levels < 1 || gray_levels > (1 << 20)) invalid("gray_levels must be in [1, 2^20]");
    cudaStream_t s = as_stream(stream);
    Scratch sc(s);
    DbcTables t = make_dbc(sc, s, side, h_ln_table, ln_len, h_weights, n_weights, gray_levels);
    FdArgs fa{};
    fa.src = d_blocks;
    fa.side = side;
    fa.n = n;
    fa.mode = FD_STACK;
    fa.clamp = clamp;
    fa.J = t.J;
    fa.smax = t.smax;
    fa.quot = t.quot;
    fa.ln = t.ln;
    fa.ln_len = t.ln_len;
    fa.w = t.w;
    fa.fd = d_fd;
    launch_fd(fa, s);
    FIC_CUDA(cudaStreamSynchronize(s));
    sc.verify("dbc");
  });
}

extern "C" int fic_dbc_v1(const uint8_t* d_blocks, int64_t n, int32_t side, int32_t clamp,
                          const double* h_ln_table, int32_t ln_len, const double* h_weights,
                          int32_t n_weights, double* d_fd, void* stream) {
  return fic_dbc_v2(d_blocks, n, side, 256, clamp, h_ln_table, ln_len, h_weights, n_weights, d_fd, stream);
}

extern "C" int fic_decode_v1(const uint8_t* d_records, int32_t height, int32_t width,
                             int32_t range_size, int32_t domain_size, int32_t stride,
                             int32_t iterations, double initial, const uint8_t* d_initial,
                             uint8_t* d_out, void* stream) {
  return guarded([&] {
    decode_impl(d_records, height, width, range_size, domain_size, stride, iterations, initial,
                d_initial, d_out, as_stream(stream));
  });
}

extern "C" int fic_decode_step_v1(const uint8_t* d_records, int32_t height, int32_t width,
                                  int32_t range_size, int32_t domain_size, int32_t stride,
                                  const double* d_src, double* d_dst, uint8_t* d_out,
                                  void* stream) {
  return guarded([&] {
    decode_step_impl(d_records, height, width, range_size, domain_size, stride, d_src, d_dst,
                     d_out, as_stream(stream));
  });
}

extern "C" int fic_shard_pack_v1(const uint8_t* d_records, const double* d_pre_rms,
                                 const double* d_post_rms, int64_t n, int64_t* d_buf, void* stream) {
  return guarded([&] {
    if (n < 0) invalid("negative range count");
    if (n == 0) return;
    k_shard_pack<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(
        d_records, d_pre_rms, d_post_rms, n, reinterpret_cast<unsigned long long*>(d_buf));
    FIC_CHECK_LAUNCH();
  });
}

extern "C" int fic_shard_unpack_v1(const int64_t* d_buf, int64_t n, uint8_t* d_records,
                                   double* d_pre_rms, double* d_post_rms, uint32_t* d_bad,
                                   void* stream) {
  return guarded([&] {
    if (n < 0) invalid("negative range count");
    FIC_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(uint32_t), as_stream(stream)));
    if (n == 0) return;
    // whole warps (the ballot), so the grid covers n rounded up to 256
    k_shard_unpack<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const unsigned long long*>(d_buf), n, d_records, d_pre_rms, d_post_rms, d_bad);
    FIC_CHECK_LAUNCH();
  });
}

extern "C" int fic_guard_selftest_v1(int32_t overrun) {
  return guarded([&] {
    if (overrun < 0 || overrun > 64) invalid("overrun must be in [0, 64]");
    cudaStream_t s = nullptr;
    Scratch sc(s);
    uint8_t* a = sc.get<uint8_t>(1000);
    uint8_t* b = sc.get<uint8_t>(1000);
    FIC_CUDA(cudaMemsetAsync(a, 1, 1000 + (size_t)(overrun > 0 ? 8 + overrun : 0), s));  // past the 16-byte tail slack
    FIC_CUDA(cudaMemsetAsync(b, 2, 1000, s));
    FIC_CUDA(cudaStreamSynchronize(s));
    sc.verify("selftest");
  });
}

extern "C" const char* fic_last_error(void) { return fic::last_error(); }
extern "C" int fic_abi_version(void) { return FIC_ABI_VERSION; }
extern "C" void fic_release(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  for (auto it = g_arenas.begin(); it != g_arenas.end();) {  // this thread's arenas on dev
    if (it->first.first == dev && !it->second.busy) {
      if (it->second.base) cudaFreeAsync(it->second.base, it->first.second);
      it = g_arenas.erase(it);
    } else {
      ++it;
    }
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
}
