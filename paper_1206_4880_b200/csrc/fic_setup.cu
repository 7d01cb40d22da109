// Setup kernels of the encoder hot path: FD (K2), slabs (K3), pool builder
// (K1), range preparation.  sm_100a.  See DESIGN.md §Kernels.
#include <cuda_fp16.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <math.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "kernels.h"

namespace fic {

// ============================================================================
// K2 — differential box counting, one thread per block.
// fdim.py:44-80: per scale s (consecutive powers of two up to smax), cell
// max/min, count = sum(floor(max/h) - floor(min/h)) + k^2, FD = sum_j
// ln(count_j) * w_j accumulated left to right (numpy's sum over <8 terms),
// clamped to [2, 3].  floor(v/h) comes from a host table built with the same
// fp64 division numpy performs, so any block side is bit-exact.
// ============================================================================

int dbc_tables(int side, uint16_t* quot, int* smax, int* ln_needed, int gray_levels) {
  std::vector<int> scales;
  for (int s = 2; s <= side / 2; s *= 2)
    if (side % s == 0) scales.push_back(s);
  int J = (int)scales.size();
  if (J < 2) return J;
  if (J > 7) invalid("block side too large for the DBC kernel (max 7 scales)");
  int need = 0;
  for (int j = 0; j < J; ++j) {
    double h = (double)(scales[j] * gray_levels) / (double)side;  // fdim.py:74 (s * gray_levels is exact)
    if (std::floor(255.0 / h) > 65535.0) invalid("gray_levels too small for this block side on the GPU path");
    for (int v = 0; v < 256; ++v) quot[j * 256 + v] = (uint16_t)std::floor((double)v / h);
    int k = side / scales[j];
    need = std::max(need, k * k * (quot[j * 256 + 255] - quot[j * 256 + 0]) + k * k);
  }
  *smax = scales.back();
  *ln_needed = need + 1;
  return J;
}

struct PixSrc {
  const uint8_t* p;
  int W, side, mode;
  __device__ __forceinline__ int operator()(int y0, int x0, int64_t b, int yy, int xx) const {
    if (mode == FD_IMAGE) return p[(int64_t)(y0 + yy) * W + x0 + xx];
    if (mode == FD_STACK) return p[b * side * side + yy * side + xx];
    const uint8_t* q = p + (int64_t)(y0 + 2 * yy) * W + x0 + 2 * xx;  // blocks.py:75-82
    return (q[0] + q[1] + q[W] + q[W + 1]) >> 2;
  }
};

template <int SMAX>
__global__ void __launch_bounds__(256) k_fd(FdArgs a) {
  constexpr int J = (SMAX == 4) ? 2 : (SMAX == 8) ? 3 : 0;
  __shared__ uint16_t quot[J][256];
  for (int i = threadIdx.x; i < J * 256; i += blockDim.x) quot[i >> 8][i & 255] = a.quot[i];
  __syncthreads();
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.n) return;
  int y0 = 0, x0 = 0;
  if (a.mode != FD_STACK) {
    int64_t by = b / a.nbx, bx = b - by * a.nbx;
    y0 = (int)by * a.bst;
    x0 = (int)bx * a.bst;
  }
  PixSrc px{a.src, a.W, a.side, a.mode};
  int cnt[J];
#pragma unroll
  for (int j = 0; j < J; ++j) cnt[j] = 0;
  const int ncell = a.side / SMAX;
  for (int cy = 0; cy < ncell; ++cy) {
    for (int cx = 0; cx < ncell; ++cx) {
      constexpr int L = SMAX / 2;
      int mx[L][L], mn[L][L];
#pragma unroll
      for (int i = 0; i < L; ++i) {
#pragma unroll
        for (int j = 0; j < L; ++j) {
          int yy = cy * SMAX + 2 * i, xx = cx * SMAX + 2 * j;
          int p0 = px(y0, x0, b, yy, xx), p1 = px(y0, x0, b, yy, xx + 1);
          int p2 = px(y0, x0, b, yy + 1, xx), p3 = px(y0, x0, b, yy + 1, xx + 1);
          mx[i][j] = max(max(p0, p1), max(p2, p3));
          mn[i][j] = min(min(p0, p1), min(p2, p3));
          cnt[0] += quot[0][mx[i][j]] - quot[0][mn[i][j]];
        }
      }
#pragma unroll
      for (int lev = 1; lev < J; ++lev) {
        const int n = L >> lev;  // cells per side at this level
#pragma unroll
        for (int i = 0; i < n; ++i) {
#pragma unroll
          for (int j = 0; j < n; ++j) {
            int a0 = max(max(mx[2 * i][2 * j], mx[2 * i][2 * j + 1]),
                         max(mx[2 * i + 1][2 * j], mx[2 * i + 1][2 * j + 1]));
            int b0 = min(min(mn[2 * i][2 * j], mn[2 * i][2 * j + 1]),
                         min(mn[2 * i + 1][2 * j], mn[2 * i + 1][2 * j + 1]));
            mx[i][j] = a0;
            mn[i][j] = b0;
            cnt[lev] += quot[lev][a0] - quot[lev][b0];
          }
        }
      }
    }
  }
  double f = 0.0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    int k = a.side >> (j + 1);
    int c = cnt[j] + k * k;
    c = min(c, a.ln_len - 1);
    double t = __dmul_rn(__ldg(a.ln + c), __ldg(a.w + j));
    f = (j == 0) ? t : __dadd_rn(f, t);
  }
  if (a.clamp) f = fmin(fmax(f, 2.0), 3.0);
  if (a.fd) a.fd[b] = f;
  if (a.key) a.key[b] = (unsigned long long)__double_as_longlong(f);
  if (a.combo || a.rank) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) c += (uint32_t)cnt[j] * (uint32_t)a.cstride[j];
    if (a.rank_of_combo) {
      const uint32_t r = __ldg(a.rank_of_combo + c);
      a.rank[b] = r;
      if (a.rank_hist) {
        atomicAdd(a.rank_hist + r, 1u);
        atomicMin(a.rank_minid + r, (uint32_t)b);
      }
    } else {
      a.combo[b] = c;
    }
  }
  if (a.iota) a.iota[b] = (uint32_t)b;
}

// K2 for 16x16 domain blocks on the image (scales 2, 4, 8) at a small
// stride: one CTA per T x T tile of domain positions.  The stride-1 domains
// overlap almost entirely, so the per-cell maxima / minima are computed once
// per pixel position of the tile's image patch (cell (y, x) of scale s covers
// pixels [y, y+s) x [x, x+s), built from scale s/2 like fdim.py:63-72), the
// per-cell count increments floor(max/h) - floor(min/h) are stored, and each
// block's count is a strided sum of them, done separably (rows, then
// columns).  Same integer counts as k_fd, hence the same FD bits.
template <int T, bool POW2>
__global__ void __launch_bounds__(256) k_fd16_tile(FdArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint16_t quot[3][256];
  for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) quot[i >> 8][i & 255] = a.quot[i];
  const int st = a.bst;
  const int PW = (T - 1) * st + 16;  // patch side (pixels)
  const int PP = PW * PW;
  uint8_t* P = sm;
  uint8_t* X2 = P + PP;
  uint8_t* N2 = X2 + PP;
  uint8_t* C2 = N2 + PP;
  uint8_t* X4 = C2 + PP;
  uint8_t* N4 = X4 + PP;
  uint8_t* C4 = N4 + PP;
  uint8_t* C8 = C4 + PP;
  uint16_t* H2 = reinterpret_cast<uint16_t*>(sm + ((8 * PP + 15) & ~15));
  uint16_t* H4 = H2 + PW * T;
  uint16_t* H8 = H4 + PW * T;
  uint32_t* hist = reinterpret_cast<uint32_t*>(H8 + PW * T + (PW * T & 1));  // [n_rank] if rank_hist
  uint32_t* minid = hist + a.n_rank;                                            // [n_rank]
  if (a.rank_hist)
    for (int r = threadIdx.x; r < a.n_rank; r += blockDim.x) {
      hist[r] = 0;
      minid[r] = 0xffffffffu;
    }
  const int64_t nby = a.n / a.nbx;
  const int kx0 = blockIdx.x * T, ky0 = blockIdx.y * T;
  const int x0 = kx0 * st, y0 = ky0 * st;
  const int Himg = (int)((nby - 1) * st + 16), Wimg = a.W;
  // 2-D loops: rows over warps, columns over lanes (no index division)
  const int wp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  auto for_xy = [&](int ny, int nx, auto&& f) {
    for (int y = wp; y < ny; y += 8)
      for (int x = ln; x < nx; x += 32) f(y, x);
  };
  // floor(v / h_j): a shift when h_j is a power of two (side 16: 32, 64, 128)
  const int sh0 = a.qshift[0], sh1 = a.qshift[1], sh2 = a.qshift[2];
  auto qd = [&](int j, int mx, int mn) -> int {
    if (POW2) {
      const int sh = j == 0 ? sh0 : (j == 1 ? sh1 : sh2);
      return (mx >> sh) - (mn >> sh);
    }
    return quot[j][mx] - quot[j][mn];
  };
  // the image patch as 4-byte words (x0 is a multiple of 32, W of 8; a word
  // never straddles the right edge), every load issued before any store
  {
    const int pw4 = (PW + 3) >> 2, nw = PW * pw4;
    constexpr int MAXW = 8;  // 76 x 19 words (stride 4) < 8 x 256
    uint32_t v[MAXW];
#pragma unroll
    for (int q = 0; q < MAXW; ++q) {
      const int i = (int)threadIdx.x + 256 * q;
      const int y = i / pw4, xw = i - y * pw4;
      const int gy = y0 + y, gx = x0 + 4 * xw;
      v[q] = (i < nw && gy < Himg && gx < Wimg)
                 ? __ldg(reinterpret_cast<const uint32_t*>(a.src + (int64_t)gy * Wimg + gx))
                 : 0u;
    }
#pragma unroll
    for (int q = 0; q < MAXW; ++q) {
      const int i = (int)threadIdx.x + 256 * q;
      if (i < nw) {
        const int y = i / pw4, xw = i - y * pw4;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (4 * xw + b < PW) P[y * PW + 4 * xw + b] = (uint8_t)(v[q] >> (8 * b));
      }
    }
  }
  __syncthreads();
  // scale 2 cells at every patch position
  for_xy(PW - 1, PW - 1, [&](int y, int x) {
    const int i = y * PW + x;
    const int p0 = P[i], p1 = P[i + 1], p2 = P[i + PW], p3 = P[i + PW + 1];
    const int mx = max(max(p0, p1), max(p2, p3)), mn = min(min(p0, p1), min(p2, p3));
    X2[i] = (uint8_t)mx;
    N2[i] = (uint8_t)mn;
    C2[i] = (uint8_t)qd(0, mx, mn);
  });
  __syncthreads();
  // scale 4 from four scale-2 cells
  for_xy(PW - 3, PW - 3, [&](int y, int x) {
    const int i = y * PW + x;
    const int mx = max(max(X2[i], X2[i + 2]), max(X2[i + 2 * PW], X2[i + 2 * PW + 2]));
    const int mn = min(min(N2[i], N2[i + 2]), min(N2[i + 2 * PW], N2[i + 2 * PW + 2]));
    X4[i] = (uint8_t)mx;
    N4[i] = (uint8_t)mn;
    C4[i] = (uint8_t)qd(1, mx, mn);
  });
  __syncthreads();
  // scale 8 from four scale-4 cells
  for_xy(PW - 7, PW - 7, [&](int y, int x) {
    const int i = y * PW + x;
    const int mx = max(max(X4[i], X4[i + 4]), max(X4[i + 4 * PW], X4[i + 4 * PW + 4]));
    const int mn = min(min(N4[i], N4[i + 4]), min(N4[i + 4 * PW], N4[i + 4 * PW + 4]));
    C8[i] = (uint8_t)qd(2, mx, mn);
  });
  __syncthreads();
  // row sums over each block's cells: H_s[y][lx] = sum_j C_s[y][lx*st + s*j]
  for (int i = threadIdx.x; i < PW * T; i += blockDim.x) {
    const int y = i / T, lx = i - (i / T) * T;
    const uint8_t* r2 = C2 + y * PW + lx * st;
    int h2 = 0, h4 = 0, h8 = 0;
    if (y < PW - 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j) h2 += r2[2 * j];
    }
    if (y < PW - 3) {
      const uint8_t* r4 = C4 + y * PW + lx * st;
#pragma unroll
      for (int j = 0; j < 4; ++j) h4 += r4[4 * j];
    }
    if (y < PW - 7) {
      const uint8_t* r8 = C8 + y * PW + lx * st;
      h8 = r8[0] + r8[8];
    }
    H2[i] = (uint16_t)h2;
    H4[i] = (uint16_t)h4;
    H8[i] = (uint16_t)h8;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < T * T; i += blockDim.x) {
    const int ly = i / T, lx = i - (i / T) * T;
    const int ky = ky0 + ly, kx = kx0 + lx;
    if (ky >= nby || kx >= a.nbx) continue;
    const int Y = ly * st;
    int cnt[3] = {0, 0, 0};
#pragma unroll
    for (int r = 0; r < 8; ++r) cnt[0] += H2[(Y + 2 * r) * T + lx];
#pragma unroll
    for (int r = 0; r < 4; ++r) cnt[1] += H4[(Y + 4 * r) * T + lx];
    cnt[2] = H8[Y * T + lx] + H8[(Y + 8) * T + lx];
    double f = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int k = 16 >> (j + 1);
      const int c = min(cnt[j] + k * k, a.ln_len - 1);
      const double t = __dmul_rn(__ldg(a.ln + c), __ldg(a.w + j));
      f = (j == 0) ? t : __dadd_rn(f, t);
    }
    if (a.clamp) f = fmin(fmax(f, 2.0), 3.0);
    const int64_t b = (int64_t)ky * a.nbx + kx;
    if (a.fd) a.fd[b] = f;
    if (a.key) a.key[b] = (unsigned long long)__double_as_longlong(f);
    if (a.combo || a.rank) {
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j) c += (uint32_t)cnt[j] * (uint32_t)a.cstride[j];
      if (a.rank_of_combo) {
        const uint32_t r = __ldg(a.rank_of_combo + c);
        a.rank[b] = r;
        if (a.rank_hist) {
          // neighbouring domains share ranks: one shared-memory update per
          // group of equal ranks in the warp (ids increase with the lane, so
          // the group's lowest lane holds its smallest id)
          const unsigned grp = __match_any_sync(__activemask(), r);
          if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) {
            atomicAdd(hist + r, (uint32_t)__popc(grp));
            atomicMin(minid + r, (uint32_t)b);
          }
        }
      } else {
        a.combo[b] = c;
      }
    }
    if (a.iota) a.iota[b] = (uint32_t)b;
  }
  if (a.rank_hist) {
    __syncthreads();
    for (int r = threadIdx.x; r < a.n_rank; r += blockDim.x)
      if (hist[r]) {
        atomicAdd(a.rank_hist + r, hist[r]);
        atomicMin(a.rank_minid + r, minid[r]);
      }
  }
}

// K2 for 16x16 domain blocks at an EVEN stride (st = 2 hs): every domain
// origin and every DBC cell corner is an even pixel position, so the cell
// maps are needed on the even sub-lattice only -- a half-resolution grid
// (y', x') = (y / 2, x / 2).  Scale-2 cells are the disjoint 2x2 blocks of
// that grid, a scale-4 cell is 2x2 neighbouring scale-2 cells, a scale-8
// cell is 2x2 scale-4 cells two half-grid steps apart (fdim.py:63-72); the
// per-block counts are the same strided sums as k_fd16_tile, on a 4x smaller
// map.  Same integer counts, hence the same FD bits.
template <int T, bool POW2>
__global__ void __launch_bounds__(256) k_fd16_half(FdArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint16_t quot[3][256];
  for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) quot[i >> 8][i & 255] = a.quot[i];
  const int hs = a.bst >> 1;          // half-grid step between domain origins
  const int HP = (T - 1) * hs + 8;    // half-grid patch side
  const int PW = 2 * HP;              // image patch side (pixels)
  const int PWP = (PW + 3) & ~3;      // patch row pitch (whole words)
  const int HH = HP * HP;
  uint8_t* P = sm;                    // [PW][PWP]
  uint8_t* X2 = P + PW * PWP;         // half-grid maps [HP][HP]
  uint8_t* N2 = X2 + HH;
  uint8_t* C2 = N2 + HH;
  uint8_t* X4 = C2 + HH;
  uint8_t* N4 = X4 + HH;
  uint8_t* C4 = N4 + HH;
  uint8_t* C8 = C4 + HH;
  uint16_t* H2 = reinterpret_cast<uint16_t*>(sm + ((PW * PWP + 7 * HH + 15) & ~15));
  uint16_t* H4 = H2 + HP * T;
  uint16_t* H8 = H4 + HP * T;
  uint32_t* hist = reinterpret_cast<uint32_t*>(H8 + HP * T + (HP * T & 1));
  uint32_t* minid = hist + a.n_rank;
  if (a.rank_hist)
    for (int r = threadIdx.x; r < a.n_rank; r += blockDim.x) {
      hist[r] = 0;
      minid[r] = 0xffffffffu;
    }
  const int64_t nby = a.n / a.nbx;
  const int kx0 = blockIdx.x * T, ky0 = blockIdx.y * T;
  const int x0 = kx0 * a.bst, y0 = ky0 * a.bst;
  const int Himg = (int)((nby - 1) * a.bst + 16), Wimg = a.W;
  const int wp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  auto for_xy = [&](int ny, int nx, auto&& f) {
    for (int y = wp; y < ny; y += 8)
      for (int x = ln; x < nx; x += 32) f(y, x);
  };
  const int sh0 = a.qshift[0], sh1 = a.qshift[1], sh2 = a.qshift[2];
  auto qd = [&](int j, int mx, int mn) -> int {
    if (POW2) {
      const int sh = j == 0 ? sh0 : (j == 1 ? sh1 : sh2);
      return (mx >> sh) - (mn >> sh);
    }
    return quot[j][mx] - quot[j][mn];
  };
  // image patch as 4-byte words (x0 = 64 hs bx: a multiple of 4; W % 4 == 0,
  // so a word starting inside the image lies inside it)
  {
    const int pw4 = PWP >> 2, nw = PW * pw4;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) {
      const int y = i / pw4, xw = i - y * pw4;
      const int gy = y0 + y, gx = x0 + 4 * xw;
      const uint32_t v = (gy < Himg && gx < Wimg)
                             ? __ldg(reinterpret_cast<const uint32_t*>(a.src + (int64_t)gy * Wimg + gx))
                             : 0u;
      *reinterpret_cast<uint32_t*>(P + y * PWP + 4 * xw) = v;
    }
  }
  __syncthreads();
  // scale 2: the disjoint 2x2 pixel blocks
  for_xy(HP, HP, [&](int y, int x) {
    const uint8_t* q = P + 2 * y * PWP + 2 * x;
    const int p0 = q[0], p1 = q[1], p2 = q[PWP], p3 = q[PWP + 1];
    const int mx = max(max(p0, p1), max(p2, p3)), mn = min(min(p0, p1), min(p2, p3));
    const int i = y * HP + x;
    X2[i] = (uint8_t)mx;
    N2[i] = (uint8_t)mn;
    C2[i] = (uint8_t)qd(0, mx, mn);
  });
  __syncthreads();
  // scale 4: 2x2 neighbouring scale-2 cells
  for_xy(HP - 1, HP - 1, [&](int y, int x) {
    const int i = y * HP + x;
    const int mx = max(max(X2[i], X2[i + 1]), max(X2[i + HP], X2[i + HP + 1]));
    const int mn = min(min(N2[i], N2[i + 1]), min(N2[i + HP], N2[i + HP + 1]));
    X4[i] = (uint8_t)mx;
    N4[i] = (uint8_t)mn;
    C4[i] = (uint8_t)qd(1, mx, mn);
  });
  __syncthreads();
  // scale 8: 2x2 scale-4 cells two half-grid steps apart
  for_xy(HP - 3, HP - 3, [&](int y, int x) {
    const int i = y * HP + x;
    const int mx = max(max(X4[i], X4[i + 2]), max(X4[i + 2 * HP], X4[i + 2 * HP + 2]));
    const int mn = min(min(N4[i], N4[i + 2]), min(N4[i + 2 * HP], N4[i + 2 * HP + 2]));
    C8[i] = (uint8_t)qd(2, mx, mn);
  });
  __syncthreads();
  // row sums per domain column: 8 scale-2, 4 scale-4, 2 scale-8 cells
  for (int i = threadIdx.x; i < HP * T; i += blockDim.x) {
    const int y = i / T, lx = i - y * T;
    const int xo = lx * hs;
    const uint8_t* r2 = C2 + y * HP + xo;
    int h2 = 0, h4 = 0, h8 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) h2 += r2[j];
    if (y < HP - 1) {
      const uint8_t* r4 = C4 + y * HP + xo;
#pragma unroll
      for (int j = 0; j < 4; ++j) h4 += r4[2 * j];
    }
    if (y < HP - 3) {
      const uint8_t* r8 = C8 + y * HP + xo;
      h8 = r8[0] + r8[4];
    }
    H2[i] = (uint16_t)h2;
    H4[i] = (uint16_t)h4;
    H8[i] = (uint16_t)h8;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < T * T; i += blockDim.x) {
    const int ly = i / T, lx = i - ly * T;
    const int ky = ky0 + ly, kx = kx0 + lx;
    if (ky >= nby || kx >= a.nbx) continue;
    const int Y = ly * hs;
    int cnt[3] = {0, 0, 0};
#pragma unroll
    for (int r = 0; r < 8; ++r) cnt[0] += H2[(Y + r) * T + lx];
#pragma unroll
    for (int r = 0; r < 4; ++r) cnt[1] += H4[(Y + 2 * r) * T + lx];
    cnt[2] = H8[Y * T + lx] + H8[(Y + 4) * T + lx];
    double f = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int k = 16 >> (j + 1);
      const int c = min(cnt[j] + k * k, a.ln_len - 1);
      const double t = __dmul_rn(__ldg(a.ln + c), __ldg(a.w + j));
      f = (j == 0) ? t : __dadd_rn(f, t);
    }
    if (a.clamp) f = fmin(fmax(f, 2.0), 3.0);
    const int64_t b = (int64_t)ky * a.nbx + kx;
    if (a.fd) a.fd[b] = f;
    if (a.key) a.key[b] = (unsigned long long)__double_as_longlong(f);
    if (a.combo || a.rank) {
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j) c += (uint32_t)cnt[j] * (uint32_t)a.cstride[j];
      if (a.rank_of_combo) {
        const uint32_t r = __ldg(a.rank_of_combo + c);
        a.rank[b] = r;
        if (a.rank_hist) {
          const unsigned grp = __match_any_sync(__activemask(), r);
          if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) {
            atomicAdd(hist + r, (uint32_t)__popc(grp));
            atomicMin(minid + r, (uint32_t)b);
          }
        }
      } else {
        a.combo[b] = c;
      }
    }
    if (a.iota) a.iota[b] = (uint32_t)b;
  }
  if (a.rank_hist) {
    __syncthreads();
    for (int r = threadIdx.x; r < a.n_rank; r += blockDim.x)
      if (hist[r]) {
        atomicAdd(a.rank_hist + r, hist[r]);
        atomicMin(a.rank_minid + r, minid[r]);
      }
  }
}

static size_t fd16_half_smem(int T, int st, int n_rank) {
  const int HP = (T - 1) * (st >> 1) + 8, PW = 2 * HP, HH = HP * HP, PWP = (PW + 3) & ~3;
  return (size_t)((PW * PWP + 7 * HH + 15) & ~15) +
         (size_t)(3 * HP * T + (HP * T & 1)) * sizeof(uint16_t) + (size_t)2 * n_rank * sizeof(uint32_t);
}

static size_t fd16_tile_smem(int T, int st, int n_rank) {
  const int PW = (T - 1) * st + 16, PP = PW * PW;
  return (size_t)((8 * PP + 15) & ~15) + (size_t)(3 * PW * T + (PW * T & 1)) * sizeof(uint16_t) +
         (size_t)2 * n_rank * sizeof(uint32_t);
}

// Generic path (coarsest scale >= 16): direct per-cell scan, slower.
__global__ void k_fd_generic(FdArgs a) {
  __shared__ uint16_t quot[7][256];
  for (int i = threadIdx.x; i < a.J * 256; i += blockDim.x) quot[i >> 8][i & 255] = a.quot[i];
  __syncthreads();
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.n) return;
  int y0 = 0, x0 = 0;
  if (a.mode != FD_STACK) {
    int64_t by = b / a.nbx, bx = b - by * a.nbx;
    y0 = (int)by * a.bst;
    x0 = (int)bx * a.bst;
  }
  PixSrc px{a.src, a.W, a.side, a.mode};
  double f = 0.0;
  for (int j = 0; j < a.J; ++j) {
    int s = 2 << j, k = a.side / s;
    int c = k * k;
    for (int cy = 0; cy < k; ++cy)
      for (int cx = 0; cx < k; ++cx) {
        int hi = 0, lo = 255;
        for (int yy = 0; yy < s; ++yy)
          for (int xx = 0; xx < s; ++xx) {
            int v = px(y0, x0, b, cy * s + yy, cx * s + xx);
            hi = max(hi, v);
            lo = min(lo, v);
          }
        c += quot[j][hi] - quot[j][lo];
      }
    c = min(c, a.ln_len - 1);
    double t = __dmul_rn(__ldg(a.ln + c), __ldg(a.w + j));
    f = (j == 0) ? t : __dadd_rn(f, t);
  }
  if (a.clamp) f = fmin(fmax(f, 2.0), 3.0);
  if (a.fd) a.fd[b] = f;
  if (a.key) a.key[b] = (unsigned long long)__double_as_longlong(f);
  if (a.iota) a.iota[b] = (uint32_t)b;
}

void launch_fd(const FdArgs& a, cudaStream_t s) {
  if (a.n == 0) return;
  int threads = 256;
  int64_t blocks = cdiv(a.n, threads);
  const bool tile_ok = a.mode == FD_IMAGE && a.side == 16 && a.J == 3 && a.smax == 8 &&
                       a.bst >= 1 && a.bst <= 4 && (a.W & 3) == 0 && !getenv("FIC_FD_DIRECT");
  if (tile_ok) {
    const int64_t nby = a.n / a.nbx;
    const int nr = a.rank_hist ? a.n_rank : 0;
    const bool pow2 = a.qshift[0] >= 0 && a.qshift[1] >= 0 && a.qshift[2] >= 0;
    {
      const int mx = (int)fd16_tile_smem(16, 4, kCountSortMaxRanks);
      smem_optin_k(k_fd16_tile<16, false>, mx);
      smem_optin_k(k_fd16_tile<32, false>, mx);
      smem_optin_k(k_fd16_tile<16, true>, mx);
      smem_optin_k(k_fd16_tile<32, true>, mx);
    }
    if (a.bst == 1) {
      constexpr int T = 32;
      dim3 grid((unsigned)cdiv(a.nbx, T), (unsigned)cdiv(nby, T));
      if (pow2)
        k_fd16_tile<T, true><<<grid, 256, fd16_tile_smem(T, 1, nr), s>>>(a);
      else
        k_fd16_tile<T, false><<<grid, 256, fd16_tile_smem(T, 1, nr), s>>>(a);
    } else if ((a.bst & 1) == 0 && !getenv("FIC_FD_FULLGRID")) {
      // even stride: the half-resolution lattice (k_fd16_half)
      constexpr int T = 32;
      const size_t smem = fd16_half_smem(T, a.bst, nr);
      smem_optin_k(k_fd16_half<T, true>, (int)fd16_half_smem(T, 4, kCountSortMaxRanks));
      smem_optin_k(k_fd16_half<T, false>, (int)fd16_half_smem(T, 4, kCountSortMaxRanks));
      dim3 grid((unsigned)cdiv(a.nbx, T), (unsigned)cdiv(nby, T));
      if (pow2)
        k_fd16_half<T, true><<<grid, 256, smem, s>>>(a);
      else
        k_fd16_half<T, false><<<grid, 256, smem, s>>>(a);
    } else {
      constexpr int T = 16;
      dim3 grid((unsigned)cdiv(a.nbx, T), (unsigned)cdiv(nby, T));
      if (pow2)
        k_fd16_tile<T, true><<<grid, 256, fd16_tile_smem(T, a.bst, nr), s>>>(a);
      else
        k_fd16_tile<T, false><<<grid, 256, fd16_tile_smem(T, a.bst, nr), s>>>(a);
    }
  } else if (a.smax == 4 && a.J == 2)
    k_fd<4><<<(unsigned)blocks, threads, 0, s>>>(a);
  else if (a.smax == 8 && a.J == 3)
    k_fd<8><<<(unsigned)blocks, threads, 0, s>>>(a);
  else
    k_fd_generic<<<(unsigned)blocks, threads, 0, s>>>(a);
  FIC_CHECK_LAUNCH();
}

// ============================================================================
// K3 — slabs.  Dynamic: [searchsorted(keys, fd - half, left),
// searchsorted(keys, fd + half, right)) (codec.py:368-370); static2: the
// midpoint split (codec.py:362-367); empty slabs fall back to the nearest
// FD (codec.py:371-375, 267-287).  Exhaustive / nosearch: codec.py:343-349.
// ============================================================================

__device__ __forceinline__ int64_t lower_bound(const double* k, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (k[m] < v) lo = m + 1; else hi = m;
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound(const double* k, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (k[m] <= v) lo = m + 1; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ int64_t upper_bound_u32(const uint32_t* k, int64_t n, uint32_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (k[m] <= v) lo = m + 1; else hi = m;
  }
  return lo;
}

// Sorted-key access: either the key array or, in rank form, a lookup of the
// rank's value; searches in rank form run over the (few) distinct values and
// map back to positions through rank_start -- the same positions, since the
// values are strictly increasing in the rank.
struct Keys {
  const SlabArgs& a;
  __device__ __forceinline__ double at(int64_t p) const {
    if (a.keys) return a.keys[p];
    // rank of position p: the last r with rank_start[r] <= p
    return a.fd_of_rank[upper_bound_u32(a.rank_start, a.n_rank + 1, (uint32_t)p) - 1];  // may be shared memory
  }
  __device__ __forceinline__ int64_t lower(double v) const {
    if (a.keys) return lower_bound(a.keys, a.D, v);
    return __ldg(a.rank_start + lower_bound(a.fd_of_rank, a.n_rank, v));
  }
  __device__ __forceinline__ int64_t upper(double v) const {
    if (a.keys) return upper_bound(a.keys, a.D, v);
    return __ldg(a.rank_start + upper_bound(a.fd_of_rank, a.n_rank, v));
  }
};

__global__ void k_slab_scalars(SlabArgs a) {
  if (threadIdx.x || blockIdx.x) return;
  Keys k{a};
  double fmn = k.at(0), fmx = k.at(a.D - 1);  // fdim.py:93-100
  a.scal[0] = fmn;
  a.scal[1] = fmx;
  if (a.strategy == FIC_STATIC2) {
    double mid = __ddiv_rn(__dadd_rn(fmn, fmx), 2.0);
    a.scal[2] = mid;
    a.scal[3] = (double)k.lower(mid);
  } else {
    a.scal[2] = a.has_delta ? a.delta : __ddiv_rn(__dsub_rn(fmx, fmn), 3.0);
    a.scal[3] = 0.0;
  }
}

__device__ int64_t nearest_fd(const Keys& k, const uint32_t* ids, int64_t n, double v) {
  // codec.py:267-287
  int64_t pos = k.lower(v);
  int64_t pl = pos > 0 ? pos - 1 : 0;
  int64_t pr = pos < n - 1 ? pos : n - 1;
  const double kl = k.at(pl), kr = k.at(pr);
  int64_t left = k.lower(kl);
  int64_t right = k.lower(kr);
  double d_lo = pos > 0 ? __dsub_rn(v, kl) : INFINITY;
  double d_hi = pos < n ? __dsub_rn(kr, v) : INFINITY;
  bool take_left = (d_lo < d_hi) || (d_lo == d_hi && ids[left] < ids[right]);
  return take_left ? left : right;
}

// rank_start[r] = first sorted position whose rank is >= r, for r in [0, n_rank]
__global__ void k_rank_start(const uint32_t* rks, int64_t D, int n_rank, uint32_t* start) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > D) return;
  const int r = p < D ? (int)rks[p] : n_rank;
  const int prev = p > 0 ? (int)rks[p - 1] : -1;
  for (int q = prev + 1; q <= r; ++q) start[q] = (uint32_t)p;
}

void launch_rank_start(const uint32_t* rks, int64_t D, int n_rank, uint32_t* start,
                       cudaStream_t s) {
  k_rank_start<<<(unsigned)cdiv(D + 1, 256), 256, 0, s>>>(rks, D, n_rank, start);
  FIC_CHECK_LAUNCH();
}

// Counting sort of the domains by FD rank: the FD kernel counted the ranks
// (rank_hist); one block turns the counts into bucket starts (= rank_start),
// then each block of the scatter reserves, per rank, a run inside the bucket
// with one global atomic and places its domains there.  Ties (equal FD) end
// up in an unspecified order -- the pools are the same sets (slabs cover
// whole runs of equal keys) and the matcher's tie rule uses the raster id,
// so the encode result does not depend on it -- except the nearest-FD
// fallback (codec.py:267-287), which takes a run's first element, the
// smallest raster index in the stable order: that one is placed first.
// The block also derives the slab scalars (k_slab_scalars) from the counts:
// f_min / f_max are the values of the first / last occupied rank
// (fdim.py:93-100), the static2 boundary is the bucket start of the first
// rank whose value is >= the midpoint.
__global__ void __launch_bounds__(1024) k_rank_scan(const uint32_t* hist, int n_rank, int64_t D,
                                                    uint32_t* start, uint32_t* cursor, ScalArgs sa) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  using Red = cub::BlockReduce<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ typename Red::TempStorage rtmp;
  __shared__ int s_first, s_last, s_lb;
  __shared__ double s_mid;
  constexpr int IPT = kCountSortMaxRanks / 1024;
  uint32_t v[IPT];
  int first = n_rank, last = -1;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int r = threadIdx.x * IPT + i;
    v[i] = r < n_rank ? hist[r] : 0u;
    if (v[i]) {
      first = min(first, r);
      last = max(last, r);
    }
  }
  first = Red(rtmp).Reduce(first, cuda::minimum<>{});
  __syncthreads();
  last = Red(rtmp).Reduce(last, cuda::maximum<>{});
  if (threadIdx.x == 0) {
    s_first = first;
    s_last = last;
  }
  Scan(tmp).ExclusiveSum(v, v);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int r = threadIdx.x * IPT + i;
    if (r < n_rank) {
      start[r] = v[i];
      cursor[r] = v[i] + 1u;  // slot v[i] holds the bucket's smallest index
    }
  }
  if (threadIdx.x == 0) start[n_rank] = (uint32_t)D;
  if (!sa.scal) return;
  __syncthreads();
  const double fmn = sa.fd_of_rank[s_first], fmx = sa.fd_of_rank[s_last];
  if (sa.strategy == FIC_STATIC2) {
    const double mid = __ddiv_rn(__dadd_rn(fmn, fmx), 2.0);
    int below = 0;  // ranks with a value < mid (values increase with the rank)
    for (int r = threadIdx.x; r < n_rank; r += blockDim.x) below += sa.fd_of_rank[r] < mid ? 1 : 0;
    below = Red(rtmp).Reduce(below, cuda::std::plus<>{});
    if (threadIdx.x == 0) {
      s_lb = below;
      s_mid = mid;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i)
      if (threadIdx.x * IPT + i == s_lb && s_lb < n_rank) sa.scal[3] = (double)v[i];
    if (threadIdx.x == 0) {
      if (s_lb >= n_rank) sa.scal[3] = (double)D;
      sa.scal[0] = fmn;
      sa.scal[1] = fmx;
      sa.scal[2] = s_mid;
    }
  } else if (threadIdx.x == 0) {
    sa.scal[0] = fmn;
    sa.scal[1] = fmx;
    sa.scal[2] = sa.has_delta ? sa.delta : __ddiv_rn(__dsub_rn(fmx, fmn), 3.0);
    sa.scal[3] = 0.0;
  }
}

__global__ void __launch_bounds__(1024) k_rank_scatter(const uint32_t* rank, int64_t D, int n_rank,
                                                       const uint32_t* minid, const uint32_t* start,
                                                       uint32_t* cursor, uint32_t* order) {
  extern __shared__ uint32_t cnt[];  // [n_rank] counts, then bases
  constexpr int IPT = 4;
  for (int r = threadIdx.x; r < n_rank; r += blockDim.x) cnt[r] = 0;
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * blockDim.x * IPT;
  uint32_t rk[IPT], loc[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t b = b0 + (int64_t)i * blockDim.x + threadIdx.x;
    rk[i] = b < D ? __ldg(rank + b) : 0xffffffffu;
    loc[i] = 0xffffffffu;
    if (b < D) {
      if ((uint32_t)b == __ldg(minid + rk[i]))
        order[__ldg(start + rk[i])] = (uint32_t)b;  // the bucket's first slot
      else
        loc[i] = atomicAdd(cnt + rk[i], 1u);
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < n_rank; r += blockDim.x)
    if (cnt[r]) cnt[r] = atomicAdd(cursor + r, cnt[r]);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t b = b0 + (int64_t)i * blockDim.x + threadIdx.x;
    if (b < D && loc[i] != 0xffffffffu) order[cnt[rk[i]] + loc[i]] = (uint32_t)b;
  }
}

void launch_count_sort(const uint32_t* rank, int64_t D, int n_rank, const uint32_t* hist,
                       const uint32_t* minid, uint32_t* start, uint32_t* cursor, uint32_t* order,
                       const ScalArgs& sa, cudaStream_t s) {
  k_rank_scan<<<1, 1024, 0, s>>>(hist, n_rank, D, start, cursor, sa);
  FIC_CHECK_LAUNCH();
  smem_optin_k(k_rank_scatter, kCountSortMaxRanks * (int)sizeof(uint32_t));
  k_rank_scatter<<<(unsigned)cdiv(D, 4096), 1024, n_rank * sizeof(uint32_t), s>>>(
      rank, D, n_rank, minid, start, cursor, order);
  FIC_CHECK_LAUNCH();
}

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  return (q * b != a && ((a < 0) != (b < 0))) ? q - 1 : q;
}

__device__ int64_t nosearch_axis(int extent, int top, int rs, int ds, int st) {
  // codec.py:434-441
  int64_t n_pos = (extent - ds) / st + 1;
  int64_t target = (int64_t)top - rs / 2;
  int64_t k0 = min(max(floordiv(target, st), (int64_t)0), n_pos - 1);
  int64_t k1 = min(max(k0 + 1, (int64_t)0), n_pos - 1);
  int64_t e1 = k1 * st - target, e0 = k0 * st - target;
  return (llabs(e1) < llabs(e0)) ? k1 : k0;
}

__global__ void k_slabs(SlabArgs a) {
  if (a.fd_of_rank && !a.keys) {  // rank form: the (few) distinct values in shared memory
    extern __shared__ double fdr[];
#pragma unroll 8
    for (int i = threadIdx.x; i < a.n_rank; i += blockDim.x) fdr[i] = __ldg(a.fd_of_rank + i);
    __syncthreads();
    a.fd_of_rank = fdr;
  }
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.R) return;
  int64_t lo, hi;
  if (a.strategy == FIC_EXHAUSTIVE) {
    lo = 0;
    hi = a.D;
  } else if (a.strategy == FIC_NOSEARCH) {
    int ry = r / a.nrx, rx = r - ry * a.nrx;
    int64_t ky = nosearch_axis(a.H, ry * a.rs, a.rs, a.ds, a.st);
    int64_t kx = nosearch_axis(a.W, rx * a.rs, a.rs, a.ds, a.st);
    lo = ky * a.ndx + kx;
    hi = lo + 1;
  } else {
    double f = a.fd_rng[r];
    if (a.strategy == FIC_STATIC2) {
      int64_t b = (int64_t)a.scal[3];
      bool below = f < a.scal[2];
      lo = below ? 0 : b;
      hi = below ? b : a.D;
    } else {
      double half = a.scal[2];
      Keys k{a};
      if (a.lo_rank) {  // rank form: keep the rank index of lo for the range sort
        const int64_t q = lower_bound(a.fd_of_rank, a.n_rank, __dsub_rn(f, half));
        lo = __ldg(a.rank_start + q);
        a.lo_rank[r] = (uint32_t)q;
      } else {
        lo = k.lower(__dsub_rn(f, half));
      }
      hi = k.upper(__dadd_rn(f, half));
    }
    if (hi <= lo) {
      lo = nearest_fd(Keys{a}, a.ids, a.D, f);
      hi = lo + 1;
      if (a.lo_rank)  // the last rank whose bucket starts at or before lo
        a.lo_rank[r] = (uint32_t)(upper_bound_u32(a.rank_start, a.n_rank + 1, (uint32_t)lo) - 1);
    }
  }
  a.lo[r] = (int32_t)lo;
  a.hi[r] = (int32_t)hi;
}

void launch_slabs(const SlabArgs& a, cudaStream_t s) {
  if ((a.strategy == FIC_STATIC2 || a.strategy == FIC_DYNAMIC_FD) && !a.scal_ready) {
    k_slab_scalars<<<1, 32, 0, s>>>(a);
    FIC_CHECK_LAUNCH();
  }
  const bool rank_form = (a.strategy == FIC_STATIC2 || a.strategy == FIC_DYNAMIC_FD) && !a.keys;
  const size_t smem = rank_form ? (size_t)a.n_rank * sizeof(double) : 0;
  smem_optin_k(k_slabs, kCountSortMaxRanks * (int)sizeof(double));
  k_slabs<<<(unsigned)cdiv(a.R, 128), 128, smem, s>>>(a);
  FIC_CHECK_LAUNCH();
}

// ============================================================================
// K1 — pool builder.  For each pool position p (FD order for dynamic_fd /
// static2, raster otherwise): the 2x2 floor-mean decimated domain
// (blocks.py:75-82) as raw bytes, its exact sums, inv_den = 1/den (0 when
// den == 0, codec.py:141-145) and the fp16 centred unit-norm row
// B_k = (K d_k - sum_d) / sqrt(K den) that the tensor-core screen consumes.
// ============================================================================

// Box-floor planes: plane[par][y][k] = (I[y][x] + I[y][x+1] + I[y+1][x] +
// I[y+1][x+1]) >> 2 with x = 2k + par.  A decimated domain row (blocks.py:
// 75-82) is then RS consecutive bytes of one plane row, so a domain is RS
// short row reads from a 2 x (H-1) x W/2 byte array that stays in L2.
__global__ void __launch_bounds__(256) k_boxplanes(const uint8_t* img, int H, int W, int pitch,
                                                   uint8_t* planes) {
  // one thread: 16 consecutive x of one row y (x0 = 16 t): rows y and y + 1
  // as five 4-byte loads each (W % 4 == 0 for 4x4 / 8x8 ranges, so x0 + 16 <
  // W implies x0 + 20 <= W), 8 outputs to each parity plane (8-byte stores)
  const int tx = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  const int x0 = 16 * tx;
  if (x0 >= W - 1 || y >= H - 1) return;
  const uint8_t* r0 = img + (int64_t)y * W + x0;
  const uint8_t* r1 = r0 + W;
  uint32_t a[5], b[5];
  const bool more = x0 + 16 < W;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const bool ok = k < 4 || more;
    a[k] = ok ? __ldg(reinterpret_cast<const uint32_t*>(r0) + k) : 0u;
    b[k] = ok ? __ldg(reinterpret_cast<const uint32_t*>(r1) + k) : 0u;
  }
  // vertical pair sums of bytes i, i+1 in 16-bit lanes, then the 2x2 sums
  uint32_t ev[4], od[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // bytes 4k .. 4k+4 of both rows
    const uint32_t lo_a = __byte_perm(a[k], 0, 0x4240), hi_a = __byte_perm(a[k], 0, 0x4341);
    const uint32_t lo_b = __byte_perm(b[k], 0, 0x4240), hi_b = __byte_perm(b[k], 0, 0x4341);
    const uint32_t nx_a = __byte_perm(a[k], a[k + 1], 0x4442), nx_b = __byte_perm(b[k], b[k + 1], 0x4442);
    const uint32_t v_e = lo_a + lo_b;   // v[4k], v[4k+2]
    const uint32_t v_o = hi_a + hi_b;   // v[4k+1], v[4k+3]
    const uint32_t v_n = __byte_perm(nx_a, 0, 0x4240) + __byte_perm(nx_b, 0, 0x4240);  // v[4k+2], v[4k+4]
    ev[k] = ((v_e + v_o) >> 2) & 0x00ff00ffu;  // x = 4k, 4k+2
    od[k] = ((v_o + v_n) >> 2) & 0x00ff00ffu;  // x = 4k+1, 4k+3
  }
  const unsigned long long e = (unsigned long long)__byte_perm(ev[0], ev[1], 0x6420) |
                               ((unsigned long long)__byte_perm(ev[2], ev[3], 0x6420) << 32);
  const unsigned long long o = (unsigned long long)__byte_perm(od[0], od[1], 0x6420) |
                               ((unsigned long long)__byte_perm(od[2], od[3], 0x6420) << 32);
  uint8_t* p0 = planes + (int64_t)y * pitch + (x0 >> 1);
  uint8_t* p1 = planes + ((int64_t)(H - 1) + y) * pitch + (x0 >> 1);
  *reinterpret_cast<unsigned long long*>(p0) = e;
  *reinterpret_cast<unsigned long long*>(p1) = o;
}

// 8 bytes starting at byte offset k of an 8-byte aligned, padded row
__device__ __forceinline__ unsigned long long bytes8(const uint8_t* row, int k) {
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(row) + (k >> 3);
  const int sh = (k & 7) * 8;
  unsigned long long lo = __ldg(w), hi = __ldg(w + 1);
  return sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
}

// One warp builds 32 consecutive pool positions: RS lanes per domain, one
// decimated row each (a short read from a box-floor plane), so every warp
// instruction moves 32/RS whole domains -- raw rows and fp16 B rows are
// stored as contiguous runs.  Row sums are reduced across the RS lanes
// (dp4a + xor shuffles) and also handed to lane j (domain p0 + j), which
// does the per-domain fp64 work once (1/den as codec.py:141-145) and writes
// the per-domain scalars coalesced.
//   B_k = fp16(fp32(K d_k - sum_d) * rsqrt(K den))
// fp32 rounding before the fp16 rounding is far inside the screen's error
// budget (fic_tc.cu: eps has 2^-12 + 2^-13 of slack beyond fp16's 2^-11).
// 8 bytes starting at byte address q (8-byte aligned loads + funnel shift)
__device__ __forceinline__ unsigned long long bytes8_at(const uint8_t* q) {
  const uintptr_t u = reinterpret_cast<uintptr_t>(q);
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(u & ~(uintptr_t)7);
  const int sh = (int)(u & 7) * 8;
  const unsigned long long lo = __ldg(w), hi = __ldg(w + 1);
  return sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
}

// Domain row segments: T[dx][y & 1][y >> 1] = the 8 box-floor values
// (I[y][x] + I[y][x+1] + I[y+1][x] + I[y+1][x+1]) >> 2 at x = X + 2j,
// j < 8, X = dx * st (blocks.py:75-82).  Row i of the domain at (Y, X) is
// T[dx][Y & 1][(Y >> 1) + i]: the pool builder reads a whole domain as 64
// contiguous bytes.  Used when T fits comfortably in L2.
// One block per 32 domain columns x 64 image rows: the image patch is staged
// in shared memory (coalesced rows), each warp computes 32 consecutive
// entries of one T[dx][par][.] run from it and writes them (256 bytes).
constexpr int DR_COLS = 32, DR_ROWS = 64;
__global__ void __launch_bounds__(256) k_domrows(const uint8_t* img, int H, int W, int st, int ndx,
                                                 int mh, unsigned long long* T) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int pw = (DR_COLS - 1) * st + 16;  // patch width (bytes)
  const int pwa = ((pw + 3) & ~3) + 4;     // row pitch: 4-byte aligned, one spare word
  uint8_t* patch = dsm;                    // [DR_ROWS + 1][pwa]
  const int dx0 = blockIdx.x * DR_COLS, y0 = blockIdx.y * DR_ROWS;
  const int X0 = dx0 * st;
  // patch rows as 4-byte words (X0 is a multiple of 32, W of 8), all loads
  // of a thread issued before any store
  const int pw4 = (pw + 3) >> 2, nw = (DR_ROWS + 1) * pw4;
  constexpr int MAXW = 12;  // words per thread for st <= 4 (65 x 36 / 256 < 10)
  if (nw <= MAXW * 256) {
    uint32_t v[MAXW];
#pragma unroll
    for (int q = 0; q < MAXW; ++q) {
      const int i = threadIdx.x + q * 256;
      const int yy = i / pw4, xw = i - yy * pw4;
      const int gy = y0 + yy, gx = X0 + 4 * xw;
      v[q] = (i < nw && gy < H && gx + 3 < W)
                 ? __ldg(reinterpret_cast<const uint32_t*>(img + (int64_t)gy * W + gx))
                 : 0u;
    }
#pragma unroll
    for (int q = 0; q < MAXW; ++q) {
      const int i = threadIdx.x + q * 256;
      if (i < nw) {
        const int yy = i / pw4, xw = i - yy * pw4;
#pragma unroll
        *reinterpret_cast<uint32_t*>(patch + yy * pwa + 4 * xw) = v[q];
      }
    }
  } else {
    for (int i = threadIdx.x; i < (DR_ROWS + 1) * pw; i += blockDim.x) {
      const int yy = i / pw, xx = i - yy * pw;
      const int gy = y0 + yy, gx = X0 + xx;
      patch[yy * pwa + xx] = (gy < H && gx < W) ? __ldg(img + (int64_t)gy * W + gx) : 0;
    }
  }
  __syncthreads();
  // lane = m within the block's 32 rows of one parity, warp-uniform (dx, par):
  // each warp writes one 256-byte run of T
  const int m0 = y0 / 2;
  for (int i = threadIdx.x; i < DR_COLS * DR_ROWS; i += blockDim.x) {
    const int ml = i % (DR_ROWS / 2), rest = i / (DR_ROWS / 2);
    const int par = rest & 1, c = rest >> 1;
    const int yy = 2 * ml + par;
    // 16 bytes of two patch rows as words (funnel-shifted to the byte
    // offset), 2x2 floor means in 16-bit lanes: (even + odd bytes) >> 2
    const int o0 = yy * pwa + c * st, sh = (o0 & 3) * 8;
    const uint32_t* q0 = reinterpret_cast<const uint32_t*>(patch + (o0 & ~3));
    const uint32_t* q1 = q0 + pwa / 4;
    uint32_t a[5], b[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      a[k] = q0[k];
      b[k] = q1[k];
    }
    uint32_t res[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t w = __funnelshift_r(a[k], a[k + 1], sh), v = __funnelshift_r(b[k], b[k + 1], sh);
      const uint32_t sum = __byte_perm(w, 0, 0x4240) + __byte_perm(w, 0, 0x4341) +
                           __byte_perm(v, 0, 0x4240) + __byte_perm(v, 0, 0x4341);
      res[k] = (sum >> 2) & 0x00ff00ffu;  // means of bytes (0,1) and (2,3) at bytes 0 and 2
    }
    unsigned long long out = (unsigned long long)__byte_perm(res[0], res[1], 0x6420) |
                             ((unsigned long long)__byte_perm(res[2], res[3], 0x6420) << 32);
    const int dx = dx0 + c, m = m0 + ml;
    if (y0 + yy >= H - 1) out = 0;
    if (dx < ndx && m < mh) T[((int64_t)dx * 2 + par) * mh + m] = out;
  }
}

// One warp builds 32 consecutive pool positions p0 .. p0 + 31.  Lane j
// locates domain p0 + j (raster id from the FD order, byte offset of its
// first decimated row in the row segments / box planes).  Per instruction
// the warp then covers DPI = 32 / RS domains, RS lanes per domain, one
// decimated row per lane: row sums by dp4a, reduced across the RS lanes,
// and the fp16 B row written as whole contiguous rows.  Lane j keeps its
// domain's sums and writes the per-domain scalars coalesced (1/den as
// codec.py:141-145: __drcp_rn(den) is the correctly rounded 1.0 / den).
//   B_k = fp16(fp32(K d_k - sum_d) * rsqrt(K den))
// fp32 rounding before the fp16 rounding is far inside the screen's error
// budget (fic_tc.cu: eps has 2^-12 + 2^-13 of slack beyond fp16's 2^-11).
template <int RS, bool TROWS, bool FULL>
__device__ __forceinline__ void pool_warp(const PoolArgs& a, int64_t p0, int lane) {
  constexpr int K = RS * RS;
  constexpr int DPI = 32 / RS;  // domains per instruction
  const int g = lane / RS, i = lane % RS;
  const uint32_t D = (uint32_t)a.D;
  const uint32_t pm = (uint32_t)p0 + lane;
  const bool mine = FULL || pm < D;
  const uint32_t my_id = mine ? (a.order ? __ldg(a.order + pm) : pm) : 0u;
  uint32_t my_off;
  {
    const uint32_t dy = my_id / (uint32_t)a.ndx, dx = my_id - dy * (uint32_t)a.ndx;
    const uint32_t Y = dy * a.st, X = dx * a.st;
    my_off = TROWS ? ((dx * 2u + (Y & 1u)) * (uint32_t)a.mh + (Y >> 1))
                   : (X & 1) * (uint32_t)a.plane_rows * (uint32_t)a.pitch + Y * (uint32_t)a.pitch + (X >> 1);
  }
  const uint32_t ip = (uint32_t)(2 * i) * (uint32_t)a.pitch;
  const unsigned long long* trow = TROWS ? a.trows + i : nullptr;
  const uint8_t* prow = TROWS ? nullptr : a.planes + ip;
  // this lane's fp16 row in the first domain it writes; +DPI domains per step
  uint16_t* bq = a.bh ? a.bh + (size_t)(p0 + g) * K + i * RS : nullptr;
  uint32_t my_sd = 0, my_sdd = 0;
  const float2 kk = make_float2((float)K, (float)K);
  // all of this lane's row loads first (memory-level parallelism: the rows
  // of 32 random domains), then the arithmetic
  unsigned long long rr[RS];
#pragma unroll
  for (int k = 0; k < RS; ++k) {
    const int dk = k * DPI + g;
    const bool ok = FULL || (uint32_t)p0 + dk < D;
    const uint32_t off = __shfl_sync(0xffffffffu, my_off, dk);
    rr[k] = 0ull;
    if (ok) rr[k] = TROWS ? __ldg(trow + off) : bytes8_at(prow + off);
  }
#pragma unroll
  for (int k = 0; k < RS; ++k) {
    const int dk = k * DPI + g;                 // domain of this lane in step k
    const bool ok = FULL || (uint32_t)p0 + dk < D;
    const unsigned long long r = rr[k];
    const uint32_t w0 = (uint32_t)r, w1 = RS == 8 ? (uint32_t)(r >> 32) : 0u;
    // row sums with byte dot products: sum x and sum x^2
    uint32_t sd = __dp4a(w0, 0x01010101u, 0u), sdd = __dp4a(w0, w0, 0u);
    if (RS == 8) {
      sd = __dp4a(w1, 0x01010101u, sd);
      sdd = __dp4a(w1, w1, sdd);
    }
#pragma unroll
    for (int m = 1; m < RS; m <<= 1) {
      sd += __shfl_xor_sync(0xffffffffu, sd, m);
      sdd += __shfl_xor_sync(0xffffffffu, sdd, m);
    }
    const int src = ((lane - k * DPI) * RS) & 31;
    const uint32_t t_sd = __shfl_sync(0xffffffffu, sd, src);
    const uint32_t t_sdd = __shfl_sync(0xffffffffu, sdd, src);
    if (lane / DPI == k) {
      my_sd = t_sd;
      my_sdd = t_sdd;
    }
    if (a.bh != nullptr && ok) {
    // x from the byte via 0x4B0000xx - 2^23 (exact), K x - sum_d by an exact
    // FMA (|.| < 2^24), packed fp32 pairs; rsqrtf's ~2 ulp are far inside the
    // screen's slack
    const int den = K * (int)sdd - (int)sd * (int)sd;  // < 2^31
    float sc = 0.0f;
    if (den > 0) {  // K den >= K: no denormal fix-up needed
      const float kd = (float)K * (float)den;
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(sc) : "f"(kd));
    }
    const float2 sc2 = make_float2(sc, sc), offs = make_float2(-(float)sd, -(float)sd);
    uint32_t h[RS / 2];
#pragma unroll
    for (int e = 0; e < RS / 2; ++e) {
      const uint32_t w = e < 2 ? w0 : w1;
      const int b0 = (2 * e) & 3;
      float2 m = make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7640 + b0)),
                             __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7640 + b0 + 1)));
      m = __fadd2_rn(m, make_float2(-8388608.0f, -8388608.0f));
      const float2 f = __fmul2_rn(__ffma2_rn(kk, m, offs), sc2);
      __half2 hv = __floats2half2_rn(f.x, f.y);
      h[e] = *reinterpret_cast<uint32_t*>(&hv);
    }
    uint16_t* dst = bq + (size_t)k * DPI * K;
    if (RS == 8)
      *reinterpret_cast<uint4*>(dst) = make_uint4(h[0], h[1], h[2], h[3]);
    else
      *reinterpret_cast<uint2*>(dst) = make_uint2(h[0], h[1]);
    }
  }
  if (mine) {
    const int64_t den = (int64_t)K * my_sdd - (int64_t)my_sd * my_sd;
    a.inv_den[pm] = den != 0 ? __drcp_rn((double)den) : 0.0;
    a.sums[pm] = make_uint2(my_sd, my_sdd);
  }
}

#ifndef FIC_POOL_BLK_T
#define FIC_POOL_BLK_T 6  // resident blocks per SM the register budget allows (row segments)
#endif
#ifndef FIC_POOL_BLK_P
#define FIC_POOL_BLK_P 6  // (box planes)
#endif
template <int RS, bool TROWS>
__global__ void __launch_bounds__(256, TROWS ? FIC_POOL_BLK_T : FIC_POOL_BLK_P) k_pool(PoolArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t p0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
  if (p0 >= a.D) return;
  // whole warps skip the per-row bounds checks (a vote keeps the branch
  // warp-uniform for the shuffles inside)
  if (__all_sync(0xffffffffu, p0 + 32 <= a.D))
    pool_warp<RS, TROWS, true>(a, p0, lane);
  else
    pool_warp<RS, TROWS, false>(a, p0, lane);
}

__global__ void k_pool_generic(PoolArgs a, int rs) {
  int K = rs * rs;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.D) return;
  uint32_t id = a.order ? a.order[p] : (uint32_t)p;
  int dy = (int)(id / (uint32_t)a.ndx), dx = (int)(id - (uint32_t)dy * a.ndx);
  const uint8_t* base = a.img + (int64_t)dy * a.st * a.W + (int64_t)dx * a.st;
  uint32_t sd = 0, sdd = 0;
  uint8_t* out = a.raw + (size_t)p * a.KP;
  for (int i = 0; i < rs; ++i)
    for (int j = 0; j < rs; ++j) {
      const uint8_t* q = base + (int64_t)(2 * i) * a.W + 2 * j;
      uint32_t x = (q[0] + q[1] + q[a.W] + q[a.W + 1]) >> 2;
      out[i * rs + j] = (uint8_t)x;
      sd += x;
      sdd += x * x;
    }
  for (int k = K; k < a.KP; ++k) out[k] = 0;  // zero padding: dp4a over whole words
  int64_t den = (int64_t)K * sdd - (int64_t)sd * sd;
  a.inv_den[p] = den != 0 ? __drcp_rn((double)den) : 0.0;
  a.sums[p] = make_uint2(sd, sdd);
}

void launch_pool(const PoolArgs& a, cudaStream_t s) {
  if (a.D == 0) return;
  unsigned blocks = (unsigned)cdiv(a.D, 256);
  if (a.rs == 8 && a.trows) {
    const int pw = (DR_COLS - 1) * a.st + 16;
    const size_t smem = (size_t)(DR_ROWS + 1) * (((pw + 3) & ~3) + 4) + 16;
    smem_optin_k(k_domrows, 200 * 1024);
    if (smem > 200 * 1024) invalid("domain stride too large for the row-segment pool builder");
    dim3 grid((unsigned)cdiv(a.ndx, DR_COLS), (unsigned)cdiv(2 * a.mh, DR_ROWS));
    k_domrows<<<grid, 256, smem, s>>>(a.img, a.H, a.W, a.st, a.ndx, a.mh, a.trows);
    FIC_CHECK_LAUNCH();
    if (a.ev_main) FIC_CUDA(record_timing_event(a.ev_main, s));
    k_pool<8, true><<<blocks, 256, 0, s>>>(a);
  } else if ((a.rs == 8 || a.rs == 4) && a.planes) {
    dim3 grid((unsigned)cdiv(cdiv(a.W - 1, 16), 256), (unsigned)(a.H - 1));
    k_boxplanes<<<grid, 256, 0, s>>>(a.img, a.H, a.W, a.pitch, a.planes);
    FIC_CHECK_LAUNCH();
    if (a.ev_main) FIC_CUDA(record_timing_event(a.ev_main, s));
    if (a.rs == 8)
      k_pool<8, false><<<blocks, 256, 0, s>>>(a);
    else
      k_pool<4, false><<<blocks, 256, 0, s>>>(a);
  } else {
    if (a.ev_main) FIC_CUDA(record_timing_event(a.ev_main, s));
    k_pool_generic<<<blocks, 256, 0, s>>>(a, a.rs);
  }
  FIC_CHECK_LAUNCH();
}

// ============================================================================
// Range preparation: sums, V, rho and the isometry-permuted range rows
// rv = r[inv_perm[iso]] (codec.py:195-198, 215, 336-337).
// ============================================================================

__global__ void k_ranges(RangeArgs a) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.R) return;
  const int rs = a.rs, K = rs * rs;
  int ry = r / a.nrx, rx = r - ry * a.nrx;
  const uint8_t* base = a.img + (int64_t)ry * rs * a.W + (int64_t)rx * rs;
  int64_t sr = 0, srr = 0;
  for (int i = 0; i < rs; ++i)
    for (int j = 0; j < rs; ++j) {
      int v = base[(int64_t)i * a.W + j];
      sr += v;
      srr += v * v;
    }
  RangeInfo inf;
  inf.sr = (double)sr;
  inf.srr = (double)srr;
  inf.V = __dsub_rn((double)srr, __ddiv_rn((double)sr * (double)sr, (double)K));
  inf.rho = (int32_t)((2 * sr + K) / (2 * K));
  inf.pad = 0;
  a.info[r] = inf;
  uint8_t* out = a.rows + (int64_t)r * a.n_iso * a.KP;
  for (int i = 0; i < a.n_iso; ++i) {
    for (int k = 0; k < K; ++k) {
      int src = a.inv_perm[i * K + k];
      out[i * a.KP + k] = base[(int64_t)(src / rs) * a.W + (src % rs)];
    }
    for (int k = K; k < a.KP; ++k) out[i * a.KP + k] = 0;
  }
}

// RS = 8 fast path: a block takes 32 ranges; their 8x8 pixels are staged
// in shared memory (one aligned 8-byte row load per thread), then one thread
// per (range, isometry) gathers its permuted row from there (no per-thread
// local-memory copy of the block).
__global__ void __launch_bounds__(256) k_ranges8(RangeArgs a) {
  __shared__ uint8_t perm[8 * 64];
  __shared__ __align__(16) uint8_t blk[32][64];
  for (int i = threadIdx.x; i < a.n_iso * 64; i += blockDim.x) perm[i] = (uint8_t)a.inv_perm[i];
  const int r0 = blockIdx.x * 32;
  {  // thread t loads row t & 7 of range r0 + (t >> 3)
    const int rl = threadIdx.x >> 3, row = threadIdx.x & 7, r = r0 + rl;
    unsigned long long v = 0ull;
    if (r < a.R) {
      const int ry = r / a.nrx, rx = r - ry * a.nrx;
      v = __ldg(reinterpret_cast<const unsigned long long*>(a.img + ((int64_t)ry * 8 + row) * a.W +
                                                            (int64_t)rx * 8));
    }
    reinterpret_cast<unsigned long long*>(blk[rl])[row] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * a.n_iso; t += blockDim.x) {
    const int rl = t / a.n_iso, iso = t - rl * a.n_iso, r = r0 + rl;
    if (r >= a.R) continue;
    const uint8_t* px = blk[rl];
    if (iso == 0) {
      int64_t sr = 0, srr = 0;
      for (int k = 0; k < 64; ++k) {
        sr += px[k];
        srr += px[k] * px[k];
      }
      RangeInfo inf;
      inf.sr = (double)sr;
      inf.srr = (double)srr;
      inf.V = __dsub_rn((double)srr, __ddiv_rn((double)sr * (double)sr, 64.0));
      inf.rho = (int32_t)((2 * sr + 64) / 128);
      inf.pad = 0;
      a.info[r] = inf;
    }
    uint4* out = reinterpret_cast<uint4*>(a.rows + ((int64_t)r * a.n_iso + iso) * 64);
    const uint8_t* pm = perm + iso * 64;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = 16 * q + 4 * e;
        w[e] = px[pm[k]] | (px[pm[k + 1]] << 8) | (px[pm[k + 2]] << 16) | ((uint32_t)px[pm[k + 3]] << 24);
      }
      out[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

void launch_ranges(const RangeArgs& a, cudaStream_t s) {
  if (a.R == 0) return;
  if (a.rs == 8 && a.W % 8 == 0) {
    k_ranges8<<<(unsigned)cdiv(a.R, 32), 256, 0, s>>>(a);
  } else {
    k_ranges<<<(unsigned)cdiv(a.R, 128), 128, 0, s>>>(a);
  }
  FIC_CHECK_LAUNCH();
}

// ============================================================================
// isometry tables (blocks.py:113-139): 0 id, 1-3 clockwise quarter turns,
// 4 fliplr, 5-7 fliplr then turns.
// ============================================================================
void iso_tables(int rs, int* perm, int* inv_perm) {
  int K = rs * rs;
  std::vector<int> cur(K), nxt(K);
  for (int i = 0; i < 8; ++i) {
    for (int k = 0; k < K; ++k) cur[k] = k;
    if (i >= 4)  // fliplr: out[y][x] = in[y][rs-1-x]
      for (int y = 0; y < rs; ++y)
        for (int x = 0; x < rs; ++x) nxt[y * rs + x] = cur[y * rs + rs - 1 - x];
    else
      nxt = cur;
    cur = nxt;
    for (int t = 0; t < i % 4; ++t) {  // clockwise: out[y][x] = in[rs-1-x][y]
      for (int y = 0; y < rs; ++y)
        for (int x = 0; x < rs; ++x) nxt[y * rs + x] = cur[(rs - 1 - x) * rs + y];
      cur = nxt;
    }
    for (int k = 0; k < K; ++k) {
      perm[i * K + k] = cur[k];
      inv_perm[i * K + cur[k]] = k;
    }
  }
}

}  // namespace fic
