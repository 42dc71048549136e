// predict.cu -- predictor-side kernels (sm_100a):
//   K5' candidate co-location sets: implicit enumeration, coarse + fine
//       predictions for many decisions (HBM-write bound)
//   K6  OLS normal-equation statistics (HBM-read bound) + 7x7 fp64 solve
//                                                   `predict.py:53-72,112-134`
//   K7  prequential SGD / RLS streams, one thread per stream `predict.py:75-205`
//   K8  EvalReport: MSE + nearest-rank relative-error quantiles
//                                                   `predict.py:176-205`
#include <math.h>

#include "capi_common.h"
#include "replay_core.cuh"

using namespace intf;

namespace {

// ===================================================================== C2
// Candidate c = (own row o, multiset of k <= cap-1 peer rows).  Per own row
// the multisets are ranked size-major (k = 0, 1, ..) and in colex order
// within a size: multiset p1<=..<=pk <-> combination c_i = p_i + (i-1) of
// {0..E+k-2}, rank = sum_i C(c_i, i).
constexpr int kMaxPeers = 7;  // cap <= 8

__host__ __device__ __forceinline__ long long binom(long long n, int k) {
  if (k < 0 || n < k) return 0;
  long long r = 1;
  for (int i = 1; i <= k; i++) r = r * (n - k + i) / i;
  return r;
}

__device__ __forceinline__ int unrank_multiset(long long r, int E, int cap, int* p) {
  int k = 0;
  for (; k < cap; k++) {
    long long nk = binom(E + k - 1, k);
    if (r < nk) break;
    r -= nk;
  }
  for (int i = k; i >= 1; i--) {
    // largest c with C(c, i) <= r, c in [i-1, E+k-2]
    int lo = i - 1, hi = E + k - 2;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (binom(mid, i) <= r) lo = mid;
      else hi = mid - 1;
    }
    r -= binom(lo, i);
    p[i - 1] = lo - (i - 1);
  }
  return k;
}

constexpr int kCandThreads = 128;
constexpr int kOwnChunk = 8;
constexpr int kMaxDec = 64;

// grid: x = multiset chunks, y = own-row chunks.  Shared: per (dec, kind, own
// in chunk) the partial fma chain over the own features, so each prediction
// is 3 fma + 1 add in fp64 (same op order as the full 6-term chain) rounded
// once to fp32.
__global__ void __launch_bounds__(kCandThreads) k_candidates(const double* __restrict__ solo,
                                                             const double* __restrict__ thr, int E, int cap,
                                                             long long n_sets, double alpha,
                                                             const double* __restrict__ coefs, int n_dec,
                                                             float* __restrict__ out) {
  __shared__ double part[kMaxDec][2][kOwnChunk];
  __shared__ double wc[kMaxDec][2][4];  // w3, w4, w5, b per (dec, kind)
  __shared__ double own_solo[kOwnChunk];
  const int o0 = blockIdx.y * kOwnChunk;
  const int no = min(kOwnChunk, E - o0);
  for (int t = threadIdx.x; t < n_dec * 2 * kOwnChunk; t += blockDim.x) {
    const int oi = t % kOwnChunk, kind = (t / kOwnChunk) & 1, d = t / (2 * kOwnChunk);
    if (oi < no) {
      const double* w = coefs + (d * 2 + kind) * 7;
      const double* x = thr + 3 * (o0 + oi);
      double acc = 0.0;
      acc = fma(w[0], x[0], acc);
      acc = fma(w[1], x[1], acc);
      acc = fma(w[2], x[2], acc);
      part[d][kind][oi] = acc;
    }
  }
  for (int t = threadIdx.x; t < n_dec * 2; t += blockDim.x) {
    const double* w = coefs + t * 7;
    wc[t >> 1][t & 1][0] = w[3];
    wc[t >> 1][t & 1][1] = w[4];
    wc[t >> 1][t & 1][2] = w[5];
    wc[t >> 1][t & 1][3] = w[6];
  }
  if (threadIdx.x < no) own_solo[threadIdx.x] = solo[o0 + threadIdx.x];
  __syncthreads();
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_sets) return;
  int p[kMaxPeers];
  const int k = unrank_multiset(r, E, cap, p);
  // colo snapshot with every peer: ((0 + p1) + p2) + ...  (`simcore.py:126-131`)
  double c0[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < k; i++) {
    c0[0] = c0[0] + thr[3 * p[i]];
    c0[1] = c0[1] + thr[3 * p[i] + 1];
    c0[2] = c0[2] + thr[3 * p[i] + 2];
  }
  // departures in (solo, row) order; snapshot i = fresh sum of the remaining
  // peers in row order; EWMA(alpha) over snapshots (`colocation.py:54-63`)
  int dep[kMaxPeers];
  bool gone[kMaxPeers];
  for (int i = 0; i < k; i++) {
    dep[i] = i;
    gone[i] = false;
  }
  for (int i = 1; i < k; i++) {  // insertion sort by (solo, row); p is row-sorted
    int v = dep[i], j = i - 1;
    while (j >= 0 && solo[p[dep[j]]] > solo[p[v]]) {
      dep[j + 1] = dep[j];
      j--;
    }
    dep[j + 1] = v;
  }
  double ew[kMaxPeers + 1][3];
  ew[0][0] = c0[0];
  ew[0][1] = c0[1];
  ew[0][2] = c0[2];
  const double om = 1.0 - alpha;
  for (int i = 1; i <= k; i++) {
    gone[dep[i - 1]] = true;
    double c[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < k; q++)
      if (!gone[q]) {
        c[0] = c[0] + thr[3 * p[q]];
        c[1] = c[1] + thr[3 * p[q] + 1];
        c[2] = c[2] + thr[3 * p[q] + 2];
      }
    for (int a = 0; a < 3; a++) ew[i][a] = alpha * c[a] + om * ew[i - 1][a];
  }
  double dep_solo[kMaxPeers];
  for (int i = 0; i < k; i++) dep_solo[i] = solo[p[dep[i]]];
  const long long ld = n_sets;  // row stride of one (dec, kind, own) slice
  for (int oi = 0; oi < no; oi++) {
    const double so = own_solo[oi];
    int j = 0;
    while (j < k && dep_solo[j] < so) j++;  // peers that finish first
    const double* f = ew[j];
    float* base = out + (long long)(o0 + oi) * ld + r;
    for (int d = 0; d < n_dec; d++) {
      const double* a = wc[d][0];
      double yc = fma(a[2], c0[2], fma(a[1], c0[1], fma(a[0], c0[0], part[d][0][oi]))) + a[3];
      const double* b = wc[d][1];
      double yf = fma(b[2], f[2], fma(b[1], f[1], fma(b[0], f[0], part[d][1][oi]))) + b[3];
      float* row = base + (long long)(d * 2) * E * ld;
      __stcs(row, (float)yc);
      __stcs(row + (long long)E * ld, (float)yf);
    }
  }
}

// ===================================================================== K6
constexpr int kOlsThreads = 256;
constexpr int kOlsBlocks = 592;  // 4 x 148 SMs
constexpr int kStats = 35;       // 28 upper-triangular G terms + 7 r terms

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kOlsThreads) k_ols_partial(const double* __restrict__ X,
                                                             const double* __restrict__ y, long long n,
                                                             double* __restrict__ ws) {
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
  for (long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (long long)gridDim.x * blockDim.x) {
    double z[7];
#pragma unroll
    for (int i = 0; i < 6; i++) z[i] = X[row * 6 + i];
    z[6] = 1.0;
    const double yy = y[row];
    int t = 0;
#pragma unroll
    for (int i = 0; i < 7; i++)
#pragma unroll
      for (int j = i; j < 7; j++) acc[t] = fma(z[i], z[j], acc[t]), t++;
#pragma unroll
    for (int i = 0; i < 7; i++) acc[28 + i] = fma(z[i], yy, acc[28 + i]);
  }
  __shared__ double red[kOlsThreads / 32][kStats];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kStats; i++) {
    double v = warp_sum(acc[i]);
    if (lane == 0) red[wid][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < kStats) {
    double v = 0.0;
    for (int w = 0; w < kOlsThreads / 32; w++) v += red[w][threadIdx.x];
    ws[(long long)blockIdx.x * kStats + threadIdx.x] = v;
  }
}

// fixed-order final reduction -> out (+=): G full 7x7 then r (deterministic)
__global__ void k_ols_final(const double* __restrict__ ws, int nblk, double* __restrict__ out) {
  const int i = threadIdx.x;
  if (i >= kStats) return;
  double v = 0.0;
  for (int b = 0; b < nblk; b++) v += ws[(long long)b * kStats + i];
  if (i < 28) {
    int t = i, r = 0;
    while (t >= 7 - r) {
      t -= 7 - r;
      r++;
    }
    const int c = r + t;
    out[r * 7 + c] += v;
    if (c != r) out[c * 7 + r] += v;
  } else {
    out[49 + (i - 28)] += v;
  }
}

// cyclic Jacobi eigenvalues of a symmetric 7x7 (fp64), for the rank test
__device__ void jacobi_eigs(const double* G, double* ev) {
  double a[7][7];
  for (int i = 0; i < 7; i++)
    for (int j = 0; j < 7; j++) a[i][j] = G[i * 7 + j];
  for (int sweep = 0; sweep < 50; sweep++) {
    double off = 0.0;
    for (int i = 0; i < 7; i++)
      for (int j = i + 1; j < 7; j++) off += a[i][j] * a[i][j];
    if (off == 0.0) break;
    for (int p = 0; p < 7; p++)
      for (int q = p + 1; q < 7; q++) {
        if (a[p][q] == 0.0) continue;
        double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 7; k++) {
          double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 7; k++) {
          double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
      }
  }
  for (int i = 0; i < 7; i++) ev[i] = a[i][i];
}

// Cholesky solve of A x = b (A SPD 7x7); returns false if not PD
__device__ bool chol_solve(const double* A, const double* b, double* x, double* inv) {
  double L[7][7];
  for (int i = 0; i < 7; i++)
    for (int j = 0; j < 7; j++) L[i][j] = 0.0;
  for (int j = 0; j < 7; j++) {
    double d = A[j * 7 + j];
    for (int k = 0; k < j; k++) d -= L[j][k] * L[j][k];
    if (!(d > 0.0)) return false;
    L[j][j] = sqrt(d);
    for (int i = j + 1; i < 7; i++) {
      double v = A[i * 7 + j];
      for (int k = 0; k < j; k++) v -= L[i][k] * L[j][k];
      L[i][j] = v / L[j][j];
    }
  }
  auto solve = [&](const double* rhs, double* out) {
    double t[7];
    for (int i = 0; i < 7; i++) {
      double v = rhs[i];
      for (int k = 0; k < i; k++) v -= L[i][k] * t[k];
      t[i] = v / L[i][i];
    }
    for (int i = 6; i >= 0; i--) {
      double v = t[i];
      for (int k = i + 1; k < 7; k++) v -= L[k][i] * out[k];
      out[i] = v / L[i][i];
    }
  };
  if (b) solve(b, x);
  if (inv) {
    for (int c = 0; c < 7; c++) {
      double e[7] = {0, 0, 0, 0, 0, 0, 0}, col[7];
      e[c] = 1.0;
      solve(e, col);
      for (int i = 0; i < 7; i++) inv[i * 7 + c] = col[i];
    }
  }
  return true;
}

// fit_ols_xy (`predict.py:53-66`): matrix_rank(Z) < 7 -> ridge solve, else
// least squares (normal equations; lstsq and Cholesky agree to ~cond*eps).
// rank test: S_i = sqrt(eig(Z^T Z)); rank = #(S_i > S_max * max(n, 7) * eps).
__global__ void k_ols_solve(const double* __restrict__ stats, double* params, int32_t* info, double* Pinv) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double G[49], r[7], ev[7];
  for (int i = 0; i < 49; i++) G[i] = stats[i];
  for (int i = 0; i < 7; i++) r[i] = stats[49 + i];
  const double n = G[48];
  jacobi_eigs(G, ev);
  double smax = 0.0;
  for (int i = 0; i < 7; i++) smax = fmax(smax, sqrt(fmax(ev[i], 0.0)));
  const double tol = smax * fmax(n, 7.0) * 2.220446049250313e-16;
  int rank = 0;
  for (int i = 0; i < 7; i++) rank += sqrt(fmax(ev[i], 0.0)) > tol;
  const bool ridge = rank < 7;
  double A[49];
  for (int i = 0; i < 49; i++) A[i] = G[i];
  if (ridge)
    for (int i = 0; i < 7; i++) A[i * 8] += 1e-8;  // RIDGE_EPS (`predict.py:18,60`)
  double x[7];
  bool ok = chol_solve(A, r, x, nullptr);
  if (!ok && !ridge) {  // numerically not PD: fall back to the ridge system
    for (int i = 0; i < 7; i++) A[i * 8] += 1e-8;
    ok = chol_solve(A, r, x, nullptr);
  }
  int fin = ok;
  for (int i = 0; i < 7; i++) {
    params[i] = ok ? x[i] : NAN;
    fin &= isfinite(x[i]);
  }
  if (info) {
    info[0] = ridge ? 1 : 0;
    info[1] = fin ? 0 : 1;
  }
  if (Pinv) {  // rls_init P0 = inv(Z^T Z), ridge on failure (`predict.py:126-131`)
    double B[49];
    for (int i = 0; i < 49; i++) B[i] = G[i];
    if (!chol_solve(B, nullptr, nullptr, Pinv)) {
      for (int i = 0; i < 7; i++) B[i * 8] += 1e-8;
      chol_solve(B, nullptr, nullptr, Pinv);
    }
  }
}

// ===================================================================== K7
// sgd_update (`predict.py:88-95`): e = y - (w.x + b); w += (eta*e)*x;
// b += eta*e -- same rounding sequence as numpy (unfused).
__global__ void k_sgd(const double* __restrict__ X, const double* __restrict__ Y, const long long* __restrict__ off,
                      int n_streams, const double* __restrict__ eta, double* params, double* pred, int32_t* status) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_streams) return;
  double w[7];
  for (int i = 0; i < 7; i++) w[i] = params[s * 7 + i];
  const double et = eta[s];
  int st = 0;
  for (long long i = off[s]; i < off[s + 1]; i++) {
    double x[6];
    for (int j = 0; j < 6; j++) x[j] = X[i * 6 + j];
    const double yh = predict7(w, x);
    pred[i] = yh;
    const double e = Y[i] - yh;
    const double ee = et * e;
    for (int j = 0; j < 6; j++) w[j] = w[j] + ee * x[j];
    w[6] = w[6] + et * e;
    bool fin = true;
    for (int j = 0; j < 7; j++) fin &= isfinite(w[j]);
    if (!fin) {
      st |= 1;  // PredictError (`predict.py:94`)
      break;
    }
  }
  for (int i = 0; i < 7; i++) params[s * 7 + i] = w[i];
  if (status) status[s] = st;
}

// rls_update (`predict.py:137-154`); P kept in registers (fully unrolled).
__global__ void __launch_bounds__(64) k_rls(const double* __restrict__ X, const double* __restrict__ Y,
                                            const long long* __restrict__ off, int n_streams,
                                            const double* __restrict__ lamv, double* params, double* Pg,
                                            double* pred, int32_t* status) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_streams) return;
  double w[7], P[49];
#pragma unroll
  for (int i = 0; i < 7; i++) w[i] = params[s * 7 + i];
#pragma unroll
  for (int i = 0; i < 49; i++) P[i] = Pg[(long long)s * 49 + i];
  const double lam = lamv[s];
  int st = 0;
  for (long long it = off[s]; it < off[s + 1]; it++) {
    double z[7];
#pragma unroll
    for (int j = 0; j < 6; j++) z[j] = X[it * 6 + j];
    z[6] = 1.0;
    const double yh = predict7(w, z);
    pred[it] = yh;
    double Pz[7];
#pragma unroll
    for (int i = 0; i < 7; i++) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < 7; j++) a = fma(P[i * 7 + j], z[j], a);
      Pz[i] = a;
    }
    double zPz = 0.0;
#pragma unroll
    for (int j = 0; j < 7; j++) zPz = fma(z[j], Pz[j], zPz);
    double denom = lam + zPz;
    if (!(denom > 0.0) || !isfinite(denom)) {  // P reset (`predict.py:142-146`)
      st |= 2;
#pragma unroll
      for (int i = 0; i < 49; i++) P[i] = (i % 8 == 0) ? 100.0 : 0.0;
#pragma unroll
      for (int i = 0; i < 7; i++) Pz[i] = 100.0 * z[i];
      zPz = 0.0;
#pragma unroll
      for (int j = 0; j < 7; j++) zPz = fma(z[j], Pz[j], zPz);
      denom = lam + zPz;
    }
    double k[7];
#pragma unroll
    for (int i = 0; i < 7; i++) k[i] = Pz[i] / denom;
    const double e = Y[it] - yh;
#pragma unroll
    for (int i = 0; i < 7; i++) w[i] = w[i] + k[i] * e;
#pragma unroll
    for (int i = 0; i < 7; i++)
#pragma unroll
      for (int j = 0; j < 7; j++) P[i * 7 + j] = (P[i * 7 + j] - k[i] * Pz[j]) / lam;
#pragma unroll
    for (int i = 0; i < 7; i++)
#pragma unroll
      for (int j = i + 1; j < 7; j++) {
        const double v = 0.5 * (P[i * 7 + j] + P[j * 7 + i]);
        P[i * 7 + j] = v;
        P[j * 7 + i] = v;
      }
    bool fin = true;
#pragma unroll
    for (int j = 0; j < 7; j++) fin &= isfinite(w[j]);
    if (!fin) {
      st |= 1;
      break;
    }
  }
#pragma unroll
  for (int i = 0; i < 7; i++) params[s * 7 + i] = w[i];
#pragma unroll
  for (int i = 0; i < 49; i++) Pg[(long long)s * 49 + i] = P[i];
  if (status) status[s] = st;
}

// ===================================================================== K8
constexpr int kEvalThreads = 256;

__device__ __forceinline__ unsigned long long f64_key(double v) {
  unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// one block per dataset: MSE (block tree sum) + 4 nearest-rank quantiles of
// rel = |yhat - y| / y by an 8-pass radix select sharing histograms.
__global__ void __launch_bounds__(kEvalThreads) k_eval(const double* __restrict__ yhat, const double* __restrict__ y,
                                                       const long long* __restrict__ off, double* __restrict__ out) {
  const int s = blockIdx.x;
  const long long a = off[s], n = off[s + 1] - off[s];
  __shared__ unsigned int hist[4][256];
  __shared__ unsigned long long prefix[4];
  __shared__ long long left[4];
  __shared__ double red[kEvalThreads / 32];
  double sq = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = yhat[a + i] - y[a + i];
    sq = fma(d, d, sq);
  }
  sq = warp_sum(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  const double pq[4] = {25.0, 50.0, 75.0, 95.0};
  if (threadIdx.x < 4) {
    long long rk = (long long)ceil((pq[threadIdx.x] / 100.0) * (double)n);
    left[threadIdx.x] = (rk < 1 ? 1 : rk) - 1;
    prefix[threadIdx.x] = 0ull;
  }
  __syncthreads();
  for (int pass = 0; pass < 8; pass++) {
    const int shift = 56 - 8 * pass;
    for (int t = threadIdx.x; t < 4 * 256; t += blockDim.x) (&hist[0][0])[t] = 0u;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      const double rel = fabs(yhat[a + i] - y[a + i]) / y[a + i];
      const unsigned long long key = f64_key(rel);
      const unsigned d = (unsigned)(key >> shift) & 0xffu;
#pragma unroll
      for (int q = 0; q < 4; q++)
        if (pass == 0 || ((key ^ prefix[q]) >> (shift + 8)) == 0ull) atomicAdd(&hist[q][d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      const int q = threadIdx.x;
      long long l = left[q];
      unsigned d = 0;
      for (; d < 255u; d++) {
        if (l < (long long)hist[q][d]) break;
        l -= hist[q][d];
      }
      left[q] = l;
      prefix[q] |= (unsigned long long)d << shift;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < kEvalThreads / 32; w++) tot += red[w];
    double* o = out + 6ll * s;
    o[0] = n ? tot / (double)n : NAN;
    for (int q = 0; q < 4; q++) o[1 + q] = n ? key_f64(prefix[q]) : NAN;
    o[5] = (double)n;
  }
}

}  // namespace

extern "C" {

int intf_candidate_count(int32_t n_rows, int32_t cap, int64_t* n_cand) {
  if (n_rows < 1 || cap < 1 || cap > kMaxPeers + 1 || !n_cand) return bad_input("intf_candidate_count: bad argument");
  long long sets = 0;
  for (int k = 0; k < cap; k++) sets += binom(n_rows + k - 1, k);
  *n_cand = (int64_t)n_rows * sets;
  return INTF_OK;
}

int intf_predict_candidates(const intf_table* table, int32_t cap, double alpha, const double* coefs, int32_t n_dec,
                            float* out, void* stream) {
  if (!table || !coefs || !out || n_dec < 1 || n_dec > kMaxDec || cap < 1 || cap > kMaxPeers + 1)
    return bad_input("intf_predict_candidates: bad argument (1 <= n_dec <= 64, 1 <= cap <= 8)");
  const int E = table->n_rows;
  long long sets = 0;
  for (int k = 0; k < cap; k++) sets += binom(E + k - 1, k);
  dim3 grid(ceil_div(sets, kCandThreads), ceil_div(E, kOwnChunk));
  k_candidates<<<grid, kCandThreads, 0, as_stream(stream)>>>(table->solo_ms, table->thr, E, cap, sets, alpha, coefs,
                                                             n_dec, out);
  return launch_status("k_candidates");
}

int intf_predict_candidates_host(const intf_table* table, int32_t cap, double alpha, const double* h_coefs,
                                 int32_t n_dec, float* h_out, float* d_scratch, void* stream) {
  if (!h_coefs || !h_out || !d_scratch) return bad_input("intf_predict_candidates_host: null argument");
  int64_t n_cand = 0;
  int rc = intf_candidate_count(table->n_rows, cap, &n_cand);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  // coefs staged at the head of the scratch buffer (doubles), outputs after it
  double* d_coefs = reinterpret_cast<double*>(d_scratch);
  float* d_out = d_scratch + 2 * (size_t)n_dec * 2 * 7;
  if (cudaMemcpyAsync(d_coefs, h_coefs, sizeof(double) * n_dec * 2 * 7, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return launch_status("copy coefs");
  rc = intf_predict_candidates(table, cap, alpha, d_coefs, n_dec, d_out, stream);
  if (rc) return rc;
  if (cudaMemcpyAsync(h_out, d_out, sizeof(float) * (size_t)n_cand * 2 * n_dec, cudaMemcpyDeviceToHost, st) !=
      cudaSuccess)
    return launch_status("copy predictions");
  return INTF_OK;
}

int intf_ols_stats(const double* X, const double* y, int64_t n, double* out, double* ws, void* stream) {
  if (!X || !y || !out || !ws || n < 0) return bad_input("intf_ols_stats: bad argument");
  cudaStream_t st = as_stream(stream);
  const int nblk = (int)((n + kOlsThreads - 1) / kOlsThreads) < kOlsBlocks ? (int)((n + kOlsThreads - 1) / kOlsThreads)
                                                                           : kOlsBlocks;
  if (nblk > 0) {
    k_ols_partial<<<nblk, kOlsThreads, 0, st>>>(X, y, (long long)n, ws);
    int rc = launch_status("k_ols_partial");
    if (rc) return rc;
  }
  k_ols_final<<<1, 64, 0, st>>>(ws, nblk, out);
  return launch_status("k_ols_final");
}

int intf_ols_solve(const double* stats, double* out_params, int32_t* out_info, double* out_Pinv, void* stream) {
  if (!stats || !out_params) return bad_input("intf_ols_solve: null argument");
  k_ols_solve<<<1, 32, 0, as_stream(stream)>>>(stats, out_params, out_info, out_Pinv);
  return launch_status("k_ols_solve");
}

int intf_sgd_streams(const double* X, const double* y, const int64_t* off, int32_t n_streams, const double* eta,
                     double* params, double* pred, int32_t* status, void* stream) {
  if (!X || !y || !off || !eta || !params || !pred || n_streams < 0) return bad_input("intf_sgd_streams: bad argument");
  if (n_streams == 0) return INTF_OK;
  k_sgd<<<ceil_div(n_streams, 64), 64, 0, as_stream(stream)>>>(X, y, (const long long*)off, n_streams, eta, params,
                                                               pred, status);
  return launch_status("k_sgd");
}

int intf_rls_streams(const double* X, const double* y, const int64_t* off, int32_t n_streams, const double* lam,
                     double* params, double* P, double* pred, int32_t* status, void* stream) {
  if (!X || !y || !off || !lam || !params || !P || !pred || n_streams < 0)
    return bad_input("intf_rls_streams: bad argument");
  if (n_streams == 0) return INTF_OK;
  k_rls<<<ceil_div(n_streams, 64), 64, 0, as_stream(stream)>>>(X, y, (const long long*)off, n_streams, lam, params, P,
                                                               pred, status);
  return launch_status("k_rls");
}

int intf_eval_report(const double* yhat, const double* y, const int64_t* off, int32_t n_seg, double* out,
                     void* stream) {
  if (!yhat || !y || !off || !out || n_seg < 0) return bad_input("intf_eval_report: bad argument");
  if (n_seg == 0) return INTF_OK;
  k_eval<<<n_seg, kEvalThreads, 0, as_stream(stream)>>>(yhat, y, (const long long*)off, out);
  return launch_status("k_eval");
}

}  // extern "C"
