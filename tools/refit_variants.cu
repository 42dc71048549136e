// refit_variants.cu -- microbenchmark (tools/, not product): windowed OLS refit
// (intf_ols_windows) decompositions on 2^24 rows (X n x 6 + y, fp64 = 940 MB).
//   v0: product fused kernel (thread per window: stats in registers + solve)
//   v1: warp-per-window stats kernel + thread-per-window solve kernel
//   v2: the solve kernel alone (statistics already in HBM)
//   v3: solve alone, fast screen (one Cholesky, L^-1, trace bound, x = L^-T L^-1 r)
//   v4: v0 with the fast solve
//   v5: warp of 32 windows, rows staged into shared memory by cp.async
//       (coalesced), thread-per-window accumulation from shared memory, fast solve
//   v7: persistent warps, one bulk copy per region of 32/Q windows, Q lanes per window
//   v8: v6 made persistent (chunk stream continues across window groups)
//   v9: v8 with TMA tensor maps (one box per chunk for X and one for y, swizzled)
//   v6: v5 with one bulk copy (cp.async.bulk + mbarrier) per lane per chunk for X and y
// Build/run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -o /tmp/rv tools/refit_variants.cu -lcuda && /tmp/rv
#include <cuda.h>
#include <cudaTypedefs.h>

#include <vector>

#include "../paper_2512_18725_b200/csrc/predict.cu"

namespace intf {
void set_last_error(const char*, ...) {}
}  // namespace intf

namespace {

// cond(G) <= trace(G) * trace(G^-1) = trace(G) * ||L^-1||_F^2
__device__ __forceinline__ void ols_solve_fast(const double* __restrict__ st, double* params, int32_t* info) {
  double G[49];
#pragma unroll
  for (int i = 0; i < 49; i++) G[i] = st[i];
  double L[7][7];
  bool full = false;
  double x[7];
  if (chol7(G, L)) {
    double d[7];
#pragma unroll
    for (int i = 0; i < 7; i++) d[i] = 1.0 / L[i][i];
    double Li[7][7];
#pragma unroll
    for (int j = 0; j < 7; j++) {
      Li[j][j] = d[j];
#pragma unroll
      for (int i = j + 1; i < 7; i++) {
        double s = 0.0;
#pragma unroll
        for (int k = j; k < i; k++) s = fma(L[i][k], Li[k][j], s);
        Li[i][j] = -s * d[i];
      }
    }
    double tr = 0.0, ti = 0.0;
#pragma unroll
    for (int i = 0; i < 7; i++) tr += G[i * 8];
#pragma unroll
    for (int i = 0; i < 7; i++)
#pragma unroll
      for (int j = 0; j <= i; j++) ti = fma(Li[i][j], Li[i][j], ti);
    full = isfinite(ti) && tr * ti < 1e10;
    if (full) {
      double t[7];
#pragma unroll
      for (int i = 0; i < 7; i++) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k <= i; k++) v = fma(Li[i][k], st[49 + k], v);
        t[i] = v;
      }
#pragma unroll
      for (int i = 0; i < 7; i++) {
        double v = 0.0;
#pragma unroll
        for (int k = i; k < 7; k++) v = fma(Li[k][i], t[k], v);
        x[i] = v;
      }
    }
  }
  if (!full) {
    int32_t inf2[2];
    ols_solve_one(st, params, inf2, nullptr);
    info[0] = inf2[0];
    info[1] = inf2[1];
    return;
  }
  int fin = 1;
#pragma unroll
  for (int i = 0; i < 7; i++) {
    params[i] = x[i];
    fin &= isfinite(x[i]);
  }
  info[0] = 0;
  info[1] = fin ? 0 : 1;
}

__global__ void k_solve_fast(const double* __restrict__ stats, long long n_win, long long n, int window,
                             double* __restrict__ params, int32_t* __restrict__ info) {
  const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_win) return;
  const long long cnt = (w + 1) * window <= n ? window : n - w * window;
  ols_solve_fast(stats + w * 56, params + w * 7, info + 3 * w);
  info[3 * w + 2] = cnt < 7 ? 1 : 0;
}

__global__ void __launch_bounds__(128) k_fused_fast(const double* __restrict__ X, const double* __restrict__ y,
                                                    long long n, int window, long long n_win,
                                                    double* __restrict__ stats, double* __restrict__ params,
                                                    int32_t* __restrict__ info) {
  const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_win) return;
  const long long lo = w * window, hi = lo + window < n ? lo + window : n;
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
#pragma unroll 4
  for (long long row = lo; row < hi; row++) {
    const double2* xr = reinterpret_cast<const double2*>(X + row * 6);
    const double2 a = __ldg(xr), b = __ldg(xr + 1), c = __ldg(xr + 2);
    const double z[7] = {a.x, a.y, b.x, b.y, c.x, c.y, 1.0};
    const double yy = __ldg(y + row);
    int t = 0;
#pragma unroll
    for (int i = 0; i < 7; i++)
#pragma unroll
      for (int j = i; j < 7; j++) acc[t] = fma(z[i], z[j], acc[t]), t++;
#pragma unroll
    for (int i = 0; i < 7; i++) acc[28 + i] = fma(z[i], yy, acc[28 + i]);
  }
  double st[56];
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++, t++) st[i * 7 + j] = st[j * 7 + i] = acc[t];
#pragma unroll
  for (int i = 0; i < 7; i++) st[49 + i] = acc[28 + i];
  if (stats) {
#pragma unroll
    for (int i = 0; i < 56; i++) stats[w * 56 + i] = st[i];
  }
  ols_solve_fast(st, params + w * 7, info + 3 * w);
  info[3 * w + 2] = hi - lo < 7 ? 1 : 0;
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// warp = 32 consecutive windows; chunk c = rows [cR, cR+R) of every window
template <int R, int WARPS, int S>
__global__ void __launch_bounds__(32 * WARPS) k_fused_async(const double* __restrict__ X, const double* __restrict__ y,
                                                            long long n, int window, long long n_win,
                                                            double* __restrict__ stats, double* __restrict__ params,
                                                            int32_t* __restrict__ info) {
  constexpr int XS = R * 7 + 1;  // per window per stage: R rows of (6 x, y), odd stride (banks)
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* buf = smem + (size_t)wid * S * 32 * XS;
  const long long w0 = ((long long)blockIdx.x * WARPS + wid) * 32;
  if (w0 >= n_win) return;
  const long long w = w0 + lane;
  const int nch = (window + R - 1) / R;
  auto issue = [&](int c) {
    double* b = buf + (c % S) * 32 * XS;
    for (int idx = lane; idx < 32 * R * 7; idx += 32) {
      const int win = idx / (R * 7), q = idx % (R * 7), r = q / 7, col = q % 7;
      const long long ww = w0 + win;
      const long long row = ww * window + (long long)c * R + r;
      if (ww < n_win && c * R + r < window && row < n)
        cp_async8(b + win * XS + q, col < 6 ? X + row * 6 + col : y + row);
    }
  };
#pragma unroll
  for (int s = 0; s < S - 1; s++) {
    if (s < nch) issue(s);
    cp_commit();
  }
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
  const long long lo = w * window, hi = lo + window < n ? lo + window : n;
  const long long cnt = w < n_win ? hi - lo : 0;
  for (int c = 0; c < nch; c++) {
    if (c + S - 1 < nch) issue(c + S - 1);
    cp_commit();
    cp_wait<S - 1>();
    __syncwarp();
    const double* b = buf + (c % S) * 32 * XS + lane * XS;
#pragma unroll
    for (int r = 0; r < R; r++) {
      if ((long long)c * R + r < cnt) {
        double z[7];
#pragma unroll
        for (int i = 0; i < 6; i++) z[i] = b[r * 7 + i];
        z[6] = 1.0;
        const double yy = b[r * 7 + 6];
        int t = 0;
#pragma unroll
        for (int i = 0; i < 7; i++)
#pragma unroll
          for (int j = i; j < 7; j++) acc[t] = fma(z[i], z[j], acc[t]), t++;
#pragma unroll
        for (int i = 0; i < 7; i++) acc[28 + i] = fma(z[i], yy, acc[28 + i]);
      }
    }
    __syncwarp();
  }
  if (w >= n_win) return;
  double st[56];
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++, t++) st[i * 7 + j] = st[j * 7 + i] = acc[t];
#pragma unroll
  for (int i = 0; i < 7; i++) st[49 + i] = acc[28 + i];
  if (stats) {
#pragma unroll
    for (int i = 0; i < 56; i++) stats[w * 56 + i] = st[i];
  }
  ols_solve_fast(st, params + w * 7, info + 3 * w);
  info[3 * w + 2] = cnt < 7 ? 1 : 0;
}

__device__ __forceinline__ void mbar_init_n(uint64_t* bar, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(cnt)
               : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_p(uint64_t* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void acc_row(double* acc, const double* z6, double yy) {
  const double z[7] = {z6[0], z6[1], z6[2], z6[3], z6[4], z6[5], 1.0};
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++) acc[t] = fma(z[i], z[j], acc[t]), t++;
#pragma unroll
  for (int i = 0; i < 7; i++) acc[28 + i] = fma(z[i], yy, acc[28 + i]);
}

// v6: warp of 32 windows (window even); chunk c = rows [cR, cR+R) of every
// window, each lane bulk-copies its window's X piece (R x 48 B) and y piece
// (R x 8 B) into its own shared slot; the last (partial) window reads global
template <int R, int WARPS, int S>
__global__ void __launch_bounds__(32 * WARPS) k_fused_bulk(const double* __restrict__ X, const double* __restrict__ y,
                                                           long long n, int window, long long n_win,
                                                           double* __restrict__ stats, double* __restrict__ params,
                                                           int32_t* __restrict__ info) {
  static_assert(R % 2 == 0, "R even");
  constexpr int XS = R * 6 + 2, YS = R + 2;  // 16-byte aligned slots; odd 16-byte strides (no bank conflicts)
  constexpr int STAGE = 32 * (XS + YS);
  extern __shared__ __align__(16) double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* base = smem + (size_t)wid * (S * STAGE + 2 * S);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + S * STAGE);
  const long long w0 = ((long long)blockIdx.x * WARPS + wid) * 32;
  if (w0 >= n_win) return;
  const long long w = w0 + lane;
  const long long lo = w * window;
  const long long cnt = w < n_win ? (lo + window < n ? window : n - lo) : 0;
  const bool bulk = cnt == window;
  const int nch = (window + R - 1) / R;
  if (lane == 0)
    for (int s = 0; s < S; s++) mbar_init_n(&bar[s], 32);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int c) {
    const int st = c % S;
    double* xs = base + st * STAGE + lane * XS;
    double* ys = base + st * STAGE + 32 * XS + lane * YS;
    const int rows = min(R, window - c * R);
    mbar_expect(&bar[st], bulk ? rows * 56u : 0u);
    if (bulk) {
      bulk_copy(xs, X + (lo + (long long)c * R) * 6, rows * 48u, &bar[st]);
      bulk_copy(ys, y + lo + (long long)c * R, rows * 8u, &bar[st]);
    }
  };
  for (int s = 0; s < S - 1 && s < nch; s++) issue(s);
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
  for (int c = 0; c < nch; c++) {
    if (c + S - 1 < nch) issue(c + S - 1);
    const int st = c % S;
    mbar_wait_p(&bar[st], (unsigned)(c / S) & 1u);
    if (bulk) {
      const double2* xs = reinterpret_cast<const double2*>(base + st * STAGE + lane * XS);
      const double2* ys = reinterpret_cast<const double2*>(base + st * STAGE + 32 * XS + lane * YS);
      const int rows = min(R, window - c * R);
      if (rows == R) {
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          const double2 a0 = xs[3 * r], a1 = xs[3 * r + 1], a2 = xs[3 * r + 2];
          const double2 b0 = xs[3 * r + 3], b1 = xs[3 * r + 4], b2 = xs[3 * r + 5];
          const double2 yy = ys[r / 2];
          const double z0[6] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y};
          const double z1[6] = {b0.x, b0.y, b1.x, b1.y, b2.x, b2.y};
          acc_row(acc, z0, yy.x);
          acc_row(acc, z1, yy.y);
        }
      } else {
        const double* xd = reinterpret_cast<const double*>(xs);
        const double* yd = reinterpret_cast<const double*>(ys);
        for (int r = 0; r < rows; r++) acc_row(acc, xd + 6 * r, yd[r]);
      }
    } else {
      for (int r = c * R; r < c * R + R && r < cnt; r++) acc_row(acc, X + (lo + r) * 6, y[lo + r]);
    }
    __syncwarp();
  }
  if (w >= n_win) return;
  double st[56];
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++, t++) st[i * 7 + j] = st[j * 7 + i] = acc[t];
#pragma unroll
  for (int i = 0; i < 7; i++) st[49 + i] = acc[28 + i];
  if (stats) {
#pragma unroll
    for (int i = 0; i < 56; i++) stats[w * 56 + i] = st[i];
  }
  ols_solve_fast(st, params + w * 7, info + 3 * w);
  info[3 * w + 2] = cnt < 7 ? 1 : 0;
}

// v7: one warp per block, persistent; a region = G = 32/Q consecutive windows
// (G*W contiguous rows) staged by ONE bulk copy for X and one for y; lane
// (g, q) accumulates rows q, q+Q, ... of window g, xor-butterfly over the Q
// lanes (deterministic), lane q == 0 solves
template <int Q, int S>
__global__ void __launch_bounds__(32) k_region(const double* __restrict__ X, const double* __restrict__ y, long long n,
                                               int window, long long n_win, double* __restrict__ stats,
                                               double* __restrict__ params, int32_t* __restrict__ info) {
  constexpr int G = 32 / Q;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x, g = lane / Q, q = lane % Q;
  const int RR = G * window;                // rows per region
  const int SX = RR * 6, SY = (RR + 1) & ~1;  // doubles per stage
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * (SX + SY));
  const long long n_reg = (n_win + G - 1) / G;
  if (lane == 0)
    for (int s = 0; s < S; s++) mbar_init_n(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto full_region = [&](long long reg) { return (reg + 1) * RR <= n; };
  auto issue = [&](long long reg, int st) {
    if (lane != 0) return;
    const bool f = full_region(reg);
    mbar_expect(&bar[st], f ? RR * 56u : 0u);
    if (f) {
      bulk_copy(smem + st * (SX + SY), X + reg * RR * 6, RR * 48u, &bar[st]);
      bulk_copy(smem + st * (SX + SY) + SX, y + reg * RR, RR * 8u, &bar[st]);
    }
  };
  const long long r0 = blockIdx.x, rs = gridDim.x;
  for (int s = 0; s < S - 1; s++)
    if (r0 + s * rs < n_reg) issue(r0 + s * rs, s);
  int k = 0;
  for (long long reg = r0; reg < n_reg; reg += rs, k++) {
    {
      const long long nxt = reg + (long long)(S - 1) * rs;
      if (nxt < n_reg) issue(nxt, (k + S - 1) % S);
    }
    const int st = k % S;
    mbar_wait_p(&bar[st], (unsigned)(k / S) & 1u);
    double acc[kStats];
#pragma unroll
    for (int i = 0; i < kStats; i++) acc[i] = 0.0;
    const long long rbase = reg * RR + (long long)g * window;
    if (full_region(reg)) {
      const double* xs = smem + st * (SX + SY) + (size_t)g * window * 6;
      const double* ys = smem + st * (SX + SY) + SX + (size_t)g * window;
#pragma unroll 2
      for (int r = q; r < window; r += Q) {
        const double2* xr = reinterpret_cast<const double2*>(xs + r * 6);
        const double2 a = xr[0], b = xr[1], c = xr[2];
        const double z6[6] = {a.x, a.y, b.x, b.y, c.x, c.y};
        acc_row(acc, z6, ys[r]);
      }
    } else {
      for (int r = q; r < window && rbase + r < n; r += Q) acc_row(acc, X + (rbase + r) * 6, y[rbase + r]);
    }
#pragma unroll
    for (int o = Q / 2; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < kStats; i++) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    const long long w = reg * G + g;
    if (q == 0 && w < n_win) {
      double st2[56];
      int t = 0;
#pragma unroll
      for (int i = 0; i < 7; i++)
#pragma unroll
        for (int j = i; j < 7; j++, t++) st2[i * 7 + j] = st2[j * 7 + i] = acc[t];
#pragma unroll
      for (int i = 0; i < 7; i++) st2[49 + i] = acc[28 + i];
      if (stats) {
#pragma unroll
        for (int i = 0; i < 56; i++) stats[w * 56 + i] = st2[i];
      }
      ols_solve_fast(st2, params + w * 7, info + 3 * w);
      const long long cnt = rbase + window <= n ? window : n - rbase;
      info[3 * w + 2] = cnt < 7 ? 1 : 0;
    }
    __syncwarp();
  }
}

// v8: v6 made persistent (one warp per block, grid = 148 x PER_SM): the chunk
// stream runs on across window groups, so the next group's first chunks are in
// flight while the lanes solve the current group
template <int R, int S>
__global__ void __launch_bounds__(32) k_bulk_persist(const double* __restrict__ X, const double* __restrict__ y,
                                                     long long n, int window, long long n_win,
                                                     double* __restrict__ stats, double* __restrict__ params,
                                                     int32_t* __restrict__ info) {
  static_assert(R % 2 == 0, "R even");
  constexpr int XS = R * 6 + 2, YS = R + 2;
  constexpr int STAGE = 32 * (XS + YS);
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  const long long n_grp = (n_win + 31) / 32;
  const int nch = (window + R - 1) / R;
  const long long g0 = blockIdx.x, gs = gridDim.x;
  const long long my_grps = g0 < n_grp ? (n_grp - 1 - g0) / gs + 1 : 0;
  const long long total = my_grps * nch;  // this warp's chunk stream
  if (lane == 0)
    for (int s = 0; s < S; s++) mbar_init_n(&bar[s], 32);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  long long i_grp = g0;  // issue cursor: group, chunk, stage
  int i_c = 0, i_st = 0;
  long long i_left = total;
  auto issue = [&]() {
    const long long w = i_grp * 32 + lane;
    const long long lo = w * window;
    const bool bulk = w < n_win && lo + window <= n;
    const int rows = min(R, window - i_c * R);
    mbar_expect(&bar[i_st], bulk ? rows * 56u : 0u);
    if (bulk) {
      bulk_copy(smem + i_st * STAGE + lane * XS, X + (lo + (long long)i_c * R) * 6, rows * 48u, &bar[i_st]);
      bulk_copy(smem + i_st * STAGE + 32 * XS + lane * YS, y + lo + (long long)i_c * R, rows * 8u, &bar[i_st]);
    }
    if (++i_c == nch) i_c = 0, i_grp += gs;
    if (++i_st == S) i_st = 0;
    i_left--;
  };
  for (int s = 0; s < S - 1 && i_left > 0; s++) issue();
  double acc[kStats];
  int st = 0;
  unsigned ph = 0;
  for (long long gi = 0; gi < my_grps; gi++) {
    const long long w = (g0 + gi * gs) * 32 + lane;
    const long long lo = w * window;
    const long long cnt = w < n_win ? (lo + window < n ? window : n - lo) : 0;
    const bool bulk = cnt == window;
#pragma unroll
    for (int i = 0; i < kStats; i++) acc[i] = 0.0;
    for (int c = 0; c < nch; c++) {
      if (i_left > 0) issue();
      mbar_wait_p(&bar[st], ph);
      if (bulk) {
        const double2* xs = reinterpret_cast<const double2*>(smem + st * STAGE + lane * XS);
        const double2* ys = reinterpret_cast<const double2*>(smem + st * STAGE + 32 * XS + lane * YS);
        const int rows = min(R, window - c * R);
        if (rows == R) {
#pragma unroll
          for (int r = 0; r < R; r += 2) {
            const double2 a0 = xs[3 * r], a1 = xs[3 * r + 1], a2 = xs[3 * r + 2];
            const double2 b0 = xs[3 * r + 3], b1 = xs[3 * r + 4], b2 = xs[3 * r + 5];
            const double2 yy = ys[r / 2];
            const double z0[6] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y};
            const double z1[6] = {b0.x, b0.y, b1.x, b1.y, b2.x, b2.y};
            acc_row(acc, z0, yy.x);
            acc_row(acc, z1, yy.y);
          }
        } else {
          const double* xd = reinterpret_cast<const double*>(xs);
          const double* yd = reinterpret_cast<const double*>(ys);
          for (int r = 0; r < rows; r++) acc_row(acc, xd + 6 * r, yd[r]);
        }
      } else {
        for (int r = c * R; r < c * R + R && r < cnt; r++) acc_row(acc, X + (lo + r) * 6, y[lo + r]);
      }
      __syncwarp();
      if (++st == S) st = 0, ph ^= 1u;
    }
    if (w < n_win) {
      double st2[56];
      int t = 0;
#pragma unroll
      for (int i = 0; i < 7; i++)
#pragma unroll
        for (int j = i; j < 7; j++, t++) st2[i * 7 + j] = st2[j * 7 + i] = acc[t];
#pragma unroll
      for (int i = 0; i < 7; i++) st2[49 + i] = acc[28 + i];
      if (stats) {
#pragma unroll
        for (int i = 0; i < 56; i++) stats[w * 56 + i] = st2[i];
      }
      ols_solve_fast(st2, params + w * 7, info + 3 * w);
      info[3 * w + 2] = cnt < 7 ? 1 : 0;
    }
  }
}

// v9: v8 with TMA tensor maps: per chunk ONE 3-D box for X ({16 doubles, 3
// groups, 32 windows}, 128-byte swizzle) and ONE 2-D box for y ({8 rows, 32
// windows}, 64-byte swizzle) instead of 64 per-lane copies; window % 8 == 0,
// R = 8.  Partial windows (and windows past the full ones) read global memory.
template <int S>
__global__ void __launch_bounds__(32) k_tma_persist(const __grid_constant__ CUtensorMap mx,
                                                    const __grid_constant__ CUtensorMap my,
                                                    const double* __restrict__ X, const double* __restrict__ y,
                                                    long long n, int window, long long n_win,
                                                    double* __restrict__ stats, double* __restrict__ params,
                                                    int32_t* __restrict__ info) {
  constexpr int R = 8;
  constexpr int XB = 32 * R * 48, YB = 32 * R * 8;  // bytes per stage
  extern __shared__ unsigned char dsm[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S * (XB + YB));
  const int lane = threadIdx.x;
  const long long n_full = n / window;  // windows staged by TMA
  const long long n_grp = (n_win + 31) / 32;
  const int nch = window / R;
  const long long g0 = blockIdx.x, gs = gridDim.x;
  const long long my_grps = g0 < n_grp ? (n_grp - 1 - g0) / gs + 1 : 0;
  if (lane == 0) {
    for (int s = 0; s < S; s++) mbar_init_n(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  long long i_grp = g0;
  int i_c = 0, i_st = 0;
  long long i_left = my_grps * nch;
  auto issue = [&]() {
    if (lane == 0) {
      const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[i_st]);
      mbar_expect(&bar[i_st], (unsigned)(XB + YB));
      const unsigned dx = (unsigned)__cvta_generic_to_shared(sm + i_st * (XB + YB));
      const unsigned dy = dx + XB;
      const int w0 = (int)(i_grp * 32);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(dx),
          "l"(&mx), "r"(0), "r"(i_c * 3), "r"(w0), "r"(b)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(dy),
          "l"(&my), "r"(i_c * R), "r"(w0), "r"(b)
          : "memory");
    }
    if (++i_c == nch) i_c = 0, i_grp += gs;
    if (++i_st == S) i_st = 0;
    i_left--;
  };
  for (int s = 0; s < S - 1 && i_left > 0; s++) issue();
  double acc[kStats];
  int st = 0;
  unsigned ph = 0;
  for (long long gi = 0; gi < my_grps; gi++) {
    const long long w = (g0 + gi * gs) * 32 + lane;
    const long long lo = w * window;
    const long long cnt = w < n_win ? (lo + window < n ? window : n - lo) : 0;
    const bool bulk = w < n_full;
#pragma unroll
    for (int i = 0; i < kStats; i++) acc[i] = 0.0;
    for (int c = 0; c < nch; c++) {
      if (i_left > 0) issue();
      mbar_wait_p(&bar[st], ph);
      if (bulk) {
        const unsigned char* xs = sm + st * (XB + YB);
        const unsigned char* ys = xs + XB;
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          double z[12];
#pragma unroll
          for (int jj = 0; jj < 6; jj++) {
            const int u = 3 * r + jj;                 // 16-byte unit in this lane's 384-byte slab
            const int rho = lane * 3 + (u >> 3);      // 128-byte row of the box
            const double2 v = *reinterpret_cast<const double2*>(xs + rho * 128 + (((u & 7) ^ (rho & 7)) << 4));
            z[2 * jj] = v.x;
            z[2 * jj + 1] = v.y;
          }
          const double2 yy =
              *reinterpret_cast<const double2*>(ys + lane * 64 + ((((r >> 1)) ^ ((lane >> 1) & 3)) << 4));
          acc_row(acc, z, yy.x);
          acc_row(acc, z + 6, yy.y);
        }
      } else {
        for (int r = c * R; r < c * R + R && r < cnt; r++) acc_row(acc, X + (lo + r) * 6, y[lo + r]);
      }
      __syncwarp();
      if (++st == S) st = 0, ph ^= 1u;
    }
    if (w < n_win) {
      double st2[56];
      int t = 0;
#pragma unroll
      for (int i = 0; i < 7; i++)
#pragma unroll
        for (int j = i; j < 7; j++, t++) st2[i * 7 + j] = st2[j * 7 + i] = acc[t];
#pragma unroll
      for (int i = 0; i < 7; i++) st2[49 + i] = acc[28 + i];
      if (stats) {
#pragma unroll
        for (int i = 0; i < 56; i++) stats[w * 56 + i] = st2[i];
      }
      ols_solve_fast(st2, params + w * 7, info + 3 * w);
      info[3 * w + 2] = cnt < 7 ? 1 : 0;
    }
  }
}

}  // namespace

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    printf("no cuTensorMapEncodeTiled\n");
    exit(1);
  }
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void k_init(double* p, long long m, unsigned long long seed) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long h = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    p[i] = (double)(h >> 11) * 0x1.0p-53;
  }
}

int main() {
  const long long n = 1ll << 24;
  double *X, *y, *st, *pr, *pr2;
  int32_t *inf, *inf2;
  CK(cudaMalloc(&X, n * 6 * 8));
  CK(cudaMalloc(&y, n * 8));
  k_init<<<1184, 256>>>(X, n * 6, 1);
  k_init<<<1184, 256>>>(y, n, 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double gb = 56.0 * n / 1e9;
  for (int W : {32, 64, 128}) {
    const long long nw = (n + W - 1) / W;
    CK(cudaMalloc(&st, nw * 56 * 8));
    CK(cudaMalloc(&pr, nw * 7 * 8));
    CK(cudaMalloc(&pr2, nw * 7 * 8));
    CK(cudaMalloc(&inf, nw * 3 * 4));
    CK(cudaMalloc(&inf2, nw * 3 * 4));
    auto timeit = [&](const char* name, auto f, double* cmp) {
      for (int i = 0; i < 3; i++) f();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int i = 0; i < 10; i++) f();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      double maxd = 0;
      if (cmp) {
        std::vector<double> a(nw * 7), b(nw * 7);
        CK(cudaMemcpy(a.data(), pr, nw * 7 * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), cmp, nw * 7 * 8, cudaMemcpyDeviceToHost));
        for (long long i = 0; i < nw * 7; i++) maxd = fmax(maxd, fabs(a[i] - b[i]) / fmax(1.0, fabs(b[i])));
      }
      printf("W=%4d %-34s %.4f ms  %7.0f GB/s (input)  %.3e fits/s  maxrel %.2e\n", W, name, ms, gb / ms * 1e3,
             nw / ms * 1e3, maxd);
    };
    auto v0 = [&] { k_ols_windows_fused<<<ceil_div(nw, 128), 128>>>(X, y, n, W, nw, st, pr2, inf2); };
    timeit("v0 fused (product)", v0, nullptr);
    auto v0n = [&] { k_ols_windows_fused<<<ceil_div(nw, 128), 128>>>(X, y, n, W, nw, nullptr, pr2, inf2); };
    timeit("v0 fused, no stats out", v0n, nullptr);
    auto v1 = [&] {
      k_ols_window_stats<<<ceil_div(nw, kWinWarps), 32 * kWinWarps>>>(X, y, n, W, nw, st);
      k_ols_window_solve<<<ceil_div(nw, 128), 128>>>(st, nw, n, W, pr, inf);
    };
    timeit("v1 warp stats + solve", v1, pr2);
    auto v1s = [&] { k_ols_window_stats<<<ceil_div(nw, kWinWarps), 32 * kWinWarps>>>(X, y, n, W, nw, st); };
    timeit("v1a warp stats only", v1s, nullptr);
    auto v2 = [&] { k_ols_window_solve<<<ceil_div(nw, 128), 128>>>(st, nw, n, W, pr, inf); };
    timeit("v2 solve only", v2, pr2);
    auto v3 = [&] { k_solve_fast<<<ceil_div(nw, 128), 128>>>(st, nw, n, W, pr, inf); };
    timeit("v3 fast solve only", v3, pr2);
    auto v4 = [&] { k_fused_fast<<<ceil_div(nw, 128), 128>>>(X, y, n, W, nw, nullptr, pr, inf); };
    timeit("v4 fused fast, no stats out", v4, pr2);
#define V5(R, WARPS, S)                                                                                   \
  {                                                                                                       \
    const int sm = WARPS * S * 32 * (R * 7 + 1) * 8;                                                      \
    CK(cudaFuncSetAttribute(k_fused_async<R, WARPS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    auto f = [&] {                                                                                        \
      k_fused_async<R, WARPS, S><<<ceil_div(nw, 32 * WARPS), 32 * WARPS, sm>>>(X, y, n, W, nw, nullptr, pr, inf); \
    };                                                                                                    \
    timeit("v5 async R" #R " warps" #WARPS " S" #S, f, pr2);                                              \
  }
    V5(4, 2, 2) V5(2, 2, 4)
#define V6(R, WARPS, S)                                                                                   \
  {                                                                                                       \
    const int sm = WARPS * (S * 32 * (R * 7 + 4) + 2 * S) * 8;                                            \
    CK(cudaFuncSetAttribute(k_fused_bulk<R, WARPS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));  \
    auto f = [&] {                                                                                        \
      k_fused_bulk<R, WARPS, S><<<ceil_div(nw, 32 * WARPS), 32 * WARPS, sm>>>(X, y, n, W, nw, nullptr, pr, inf); \
    };                                                                                                    \
    timeit("v6 bulk R" #R " warps" #WARPS " S" #S, f, pr2);                                               \
  }
    V6(8, 2, 2) V6(16, 1, 2)
#define V7(Q, S, PER_SM)                                                                                  \
  {                                                                                                       \
    const int RR = 32 / Q * W;                                                                            \
    const int sm = (S * (RR * 6 + ((RR + 1) & ~1)) + S) * 8;                                              \
    CK(cudaFuncSetAttribute(k_region<Q, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));            \
    auto f = [&] { k_region<Q, S><<<148 * PER_SM, 32, sm>>>(X, y, n, W, nw, nullptr, pr, inf); };         \
    char nm[64];                                                                                          \
    snprintf(nm, sizeof nm, "v7 region Q%d S%d x%d (%d KB)", Q, S, PER_SM, sm / 1024);                    \
    timeit(nm, f, pr2);                                                                                   \
  }
    V7(4, 2, 3)
#define V8(R, S, PER_SM)                                                                                  \
  {                                                                                                       \
    const int sm = (S * 32 * (R * 7 + 4) + S) * 8;                                                        \
    CK(cudaFuncSetAttribute(k_bulk_persist<R, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));      \
    auto f = [&] { k_bulk_persist<R, S><<<148 * PER_SM, 32, sm>>>(X, y, n, W, nw, nullptr, pr, inf); };   \
    char nm[64];                                                                                          \
    snprintf(nm, sizeof nm, "v8 persist R%d S%d x%d (%d KB)", R, S, PER_SM, sm / 1024);                   \
    timeit(nm, f, pr2);                                                                                   \
  }
    V8(8, 2, 7)
    {
      static PFN_cuTensorMapEncodeTiled_v12000 enc = get_encode();
      CUtensorMap mx, my;
      const long long nf = n / W;
      cuuint64_t dx[3] = {16, (cuuint64_t)(W * 6 / 16), (cuuint64_t)nf}, sx[2] = {128, (cuuint64_t)W * 48};
      cuuint32_t bx[3] = {16, 3, 32}, ex[3] = {1, 1, 1};
      CUresult r1 = enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, dx, sx, bx, ex, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cuuint64_t dy[2] = {(cuuint64_t)W, (cuuint64_t)nf}, sy[1] = {(cuuint64_t)W * 8};
      cuuint32_t by[2] = {8, 32}, ey[2] = {1, 1};
      CUresult r2 = enc(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, y, dy, sy, by, ey, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r1 || r2) printf("encode failed %d %d\n", (int)r1, (int)r2);
#define V9(S, PER_SM)                                                                                     \
  {                                                                                                       \
    const int sm = S * 32 * 8 * 56 + 1024 + 64;                                                           \
    CK(cudaFuncSetAttribute(k_tma_persist<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));          \
    auto f = [&] { k_tma_persist<S><<<148 * PER_SM, 32, sm>>>(mx, my, X, y, n, W, nw, nullptr, pr, inf); }; \
    char nm[64];                                                                                          \
    snprintf(nm, sizeof nm, "v9 tma S%d x%d (%d KB)", S, PER_SM, sm / 1024);                              \
    timeit(nm, f, pr2);                                                                                   \
  }
      V9(2, 7) V9(3, 5) V9(4, 3) V9(2, 4) V9(3, 4) V9(6, 2) V9(8, 2)
    }
    CK(cudaGetLastError());
    cudaFree(st);
    cudaFree(pr);
    cudaFree(pr2);
    cudaFree(inf);
    cudaFree(inf2);
  }
  return 0;
}
