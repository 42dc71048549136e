// rows.cu -- array-level entry points behind the per-object reference API
// (`colocation.py:95-105` samples_from_outcomes over arbitrary outcome lists,
// `predict.py:43-44` predict over rows, `metrics.py:28-36,49-79` percentile
// and slo_report over record lists).  Same arithmetic as replay.cu/predict.cu.
#include <math.h>
#include <string.h>

#include "capi_common.h"
#include "replay_core.cuh"

using namespace intf;

namespace {

constexpr int kMaxPredRows = 8;
struct PredRowsBlock {
  intf_predictor p[kMaxPredRows];
};

// one thread per outcome row: features (static / EWMA over its colo history)
// + predictions, and the interference ratio y = measured / profiled.
__global__ void k_features_rows(const double* __restrict__ own, const int64_t* __restrict__ seg_off,
                                const int32_t* __restrict__ nseg, const double* __restrict__ colo,
                                const double* __restrict__ measured, const double* __restrict__ profiled, long long n,
                                PredRowsBlock P, int n_pred, double* __restrict__ X, double* __restrict__ Y,
                                double* __restrict__ Yhat) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double o[3] = {own[3 * i], own[3 * i + 1], own[3 * i + 2]};
  const double* h = colo + 3 * seg_off[i];
  const int ns = nseg[i];
  if (Y) Y[i] = measured[i] / profiled[i];
  for (int p = 0; p < n_pred; p++) {
    double x[6];
    features_one(o, h, ns, P.p[p].ewma, P.p[p].alpha, x);
    if (X) {
      double* xo = X + (p * n + i) * 6;
#pragma unroll
      for (int k = 0; k < 6; k++) xo[k] = x[k];
    }
    if (Yhat) Yhat[p * n + i] = predict7(P.p[p].w, x);
  }
}

// predict (`predict.py:43-44`) for rows X[n][6] under one model w[7]
__global__ void k_predict_rows(const double* __restrict__ X, long long n, const double* __restrict__ w,
                               double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[6];
#pragma unroll
  for (int k = 0; k < 6; k++) x[k] = X[i * 6 + k];
  double wl[7];
#pragma unroll
  for (int k = 0; k < 7; k++) wl[k] = w[k];
  out[i] = predict7(wl, x);
}

// ---- block radix select of up to kMaxQ nearest-rank order statistics
constexpr int kSelThreads = 256;
constexpr int kMaxQ = 8;

__device__ __forceinline__ unsigned long long okey(double v) {
  unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// values[0..n): ranks[q] (0-based) -> out[q]
__global__ void __launch_bounds__(kSelThreads) k_quantiles(const double* __restrict__ v, long long n,
                                                           const double* __restrict__ ps, int nq,
                                                           double* __restrict__ out) {
  __shared__ unsigned int hist[kMaxQ][256];
  __shared__ unsigned long long prefix[kMaxQ];
  __shared__ long long left[kMaxQ];
  if (threadIdx.x < nq) {
    // nearest rank: max(1, ceil(p/100 * n)) (`metrics.py:35`)
    long long rk = (long long)ceil((ps[threadIdx.x] / 100.0) * (double)n);
    left[threadIdx.x] = (rk < 1 ? 1 : rk) - 1;
    prefix[threadIdx.x] = 0ull;
  }
  __syncthreads();
  for (int pass = 0; pass < 8; pass++) {
    const int shift = 56 - 8 * pass;
    for (int t = threadIdx.x; t < kMaxQ * 256; t += blockDim.x) (&hist[0][0])[t] = 0u;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long key = okey(v[i]);
      const unsigned d = (unsigned)(key >> shift) & 0xffu;
      for (int q = 0; q < nq; q++)
        if (pass == 0 || ((key ^ prefix[q]) >> (shift + 8)) == 0ull) atomicAdd(&hist[q][d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < nq) {
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
  if (threadIdx.x < nq) out[threadIdx.x] = okey_inv(prefix[threadIdx.x]);
}

// slo_report over record arrays: per group (model) n, met and p50/95/99 of
// latency = completion - arrival for records with arrival >= cutoff.
__global__ void __launch_bounds__(kSelThreads) k_latency_report(const int32_t* __restrict__ grp,
                                                                const double* __restrict__ arrival,
                                                                const double* __restrict__ completion,
                                                                const uint8_t* __restrict__ met, long long n,
                                                                double cutoff, int32_t* out_n, int32_t* out_met,
                                                                double* out_p) {
  const int g = blockIdx.x;  // one block per group
  __shared__ unsigned int hist[3][256];
  __shared__ unsigned long long prefix[3];
  __shared__ long long left[3];
  __shared__ int cn, cm;
  if (threadIdx.x == 0) cn = cm = 0;
  __syncthreads();
  for (long long i = threadIdx.x; i < n; i += blockDim.x)
    if (grp[i] == g && arrival[i] >= cutoff) {
      atomicAdd(&cn, 1);
      atomicAdd(&cm, met[i] ? 1 : 0);
    }
  __syncthreads();
  const double pq[3] = {50.0, 95.0, 99.0};
  if (threadIdx.x < 3) {
    long long rk = (long long)ceil((pq[threadIdx.x] / 100.0) * (double)cn);
    left[threadIdx.x] = (rk < 1 ? 1 : rk) - 1;
    prefix[threadIdx.x] = 0ull;
  }
  __syncthreads();
  for (int pass = 0; pass < 8; pass++) {
    const int shift = 56 - 8 * pass;
    for (int t = threadIdx.x; t < 3 * 256; t += blockDim.x) (&hist[0][0])[t] = 0u;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      if (grp[i] != g || !(arrival[i] >= cutoff)) continue;
      const unsigned long long key = okey(completion[i] - arrival[i]);
      const unsigned d = (unsigned)(key >> shift) & 0xffu;
      for (int q = 0; q < 3; q++)
        if (pass == 0 || ((key ^ prefix[q]) >> (shift + 8)) == 0ull) atomicAdd(&hist[q][d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 3) {
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
    out_n[g] = cn;
    out_met[g] = cm;
  }
  if (threadIdx.x < 3) out_p[3 * g + threadIdx.x] = cn ? okey_inv(prefix[threadIdx.x]) : NAN;
}

// InterferenceOracle.noise_draw (`oracle.py:24-33`) for n (batch, segment) keys
__global__ void k_noise(unsigned long long seed, double sigma, const int64_t* __restrict__ batch,
                        const int64_t* __restrict__ seg, long long n, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = noise_draw(seed, (uint64_t)batch[i], (uint64_t)seg[i], sigma);
}

// oracle_slowdown (`oracle.py:36-47`) for n (own, colo, noise) rows
__global__ void k_slowdowns(const double* __restrict__ own, const double* __restrict__ colo, double b0, double b1,
                            double b2, const double* __restrict__ noise, long long n, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double o[3] = {own[3 * i], own[3 * i + 1], own[3 * i + 2]};
  const double c[3] = {colo[3 * i], colo[3 * i + 1], colo[3 * i + 2]};
  const double beta[3] = {b0, b1, b2};
  out[i] = slowdown(o, c, beta, noise ? noise[i] : 1.0);
}

// one PCG64 stream seeded from SeedSequence(words): n standard normals
// (numpy Generator.standard_normal), serial in one thread.
__global__ void k_normals(const uint32_t* __restrict__ words, int nw, long long n, int uniform,
                          double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t w[8];
  for (int i = 0; i < nw && i < 8; i++) w[i] = words[i];
  Pcg64 g = pcg_seed_words(w, nw < 8 ? nw : 8);
  for (long long i = 0; i < n; i++) out[i] = uniform ? pcg_next_double(g) : zig_normal(g);
}

// ---- scalar calls of the per-object API (one value per call: a hand-driven
// GpuState's reseat, a per-sample learner update, ...): the arguments travel
// as kernel parameters (bit patterns) and the results land in mapped pinned
// host memory, so a call is one launch + one stream synchronisation instead
// of tensor allocations and copies.  Same device functions / operation order
// as the batched kernels, so a scalar result equals its batched twin.
struct ScalarArgs {
  unsigned long long u[72];
};

__device__ __forceinline__ double dbits(unsigned long long v) { return __longlong_as_double((long long)v); }

__global__ void k_scalar(int op, ScalarArgs a, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  switch (op) {
    case INTF_SCALAR_NOISE:  // (seed, batch, seg, sigma) -> noise (`oracle.py:24-33`)
      out[0] = noise_draw(a.u[0], a.u[1], a.u[2], dbits(a.u[3]));
      break;
    case INTF_SCALAR_SLOWDOWN: {  // (own3, colo3, beta3, noise) -> slowdown (`oracle.py:36-47`)
      double o[3], c[3], b[3];
      for (int i = 0; i < 3; i++) o[i] = dbits(a.u[i]), c[i] = dbits(a.u[3 + i]), b[i] = dbits(a.u[6 + i]);
      out[0] = slowdown(o, c, b, dbits(a.u[9]));
      break;
    }
    case INTF_SCALAR_PREDICT: {  // (w7, x6) -> w.x + b (`predict.py:43-44`)
      double w[7], x[6];
      for (int i = 0; i < 7; i++) w[i] = dbits(a.u[i]);
      for (int i = 0; i < 6; i++) x[i] = dbits(a.u[7 + i]);
      out[0] = predict7(w, x);
      break;
    }
    case INTF_SCALAR_EWMA: {  // (r3, x3, alpha) -> alpha x + (1 - alpha) r (`colocation.py:61`)
      const double al = dbits(a.u[6]), om = 1.0 - al;
      for (int i = 0; i < 3; i++) out[i] = al * dbits(a.u[3 + i]) + om * dbits(a.u[i]);
      break;
    }
    case INTF_SCALAR_SGD: {  // (w7, x6, y, eta) -> (w7', yhat, status) as k_sgd (`predict.py:88-95`)
      double w[7], x[6];
      for (int i = 0; i < 7; i++) w[i] = dbits(a.u[i]);
      for (int i = 0; i < 6; i++) x[i] = dbits(a.u[7 + i]);
      const double y = dbits(a.u[13]), et = dbits(a.u[14]);
      const double yh = predict7(w, x);
      const double e = y - yh, ee = et * e;
      for (int j = 0; j < 6; j++) w[j] = w[j] + ee * x[j];
      w[6] = w[6] + et * e;
      bool fin = true;
      for (int j = 0; j < 7; j++) fin &= isfinite(w[j]);
      for (int j = 0; j < 7; j++) out[j] = w[j];
      out[7] = yh;
      out[8] = fin ? 0.0 : 1.0;
      break;
    }
    case INTF_SCALAR_RLS: {  // (w7, P49, x6, y, lam) -> (w7', P49', yhat, status) as k_rls_g8 (`predict.py:137-154`)
      double w[7], P[49], z[7], Pz[7], k[7];
      for (int i = 0; i < 7; i++) w[i] = dbits(a.u[i]);
      for (int i = 0; i < 49; i++) P[i] = dbits(a.u[7 + i]);
      for (int i = 0; i < 6; i++) z[i] = dbits(a.u[56 + i]);
      z[6] = 1.0;
      const double y = dbits(a.u[62]), lam = dbits(a.u[63]), inv_lam = 1.0 / lam;
      const double yh = predict7(w, z);
      bool sym = true;  // as k_rls_g8: an exactly symmetric P takes the symmetric update, no symmetrization
      for (int r = 0; r < 7; r++)
        for (int j = 0; j < 7; j++) sym &= P[r * 7 + j] == P[j * 7 + r];
      for (int r = 0; r < 7; r++) {
        double acc = 0.0;
        for (int j = 0; j < 7; j++) acc = fma(P[r * 7 + j], z[j], acc);
        Pz[r] = acc;
      }
      double zPz = 0.0;
      for (int j = 0; j < 7; j++) zPz = fma(z[j], Pz[j], zPz);
      double denom = lam + zPz;
      int st = 0;
      if (!(denom > 0.0) || !isfinite(denom)) {  // P reset (`predict.py:142-146`)
        st |= 2;
        double zr = 0.0;
        for (int j = 0; j < 7; j++) zr = fma(z[j], 100.0 * z[j], zr);
        for (int i = 0; i < 49; i++) P[i] = (i % 8 == 0) ? 100.0 : 0.0;
        for (int j = 0; j < 7; j++) Pz[j] = 100.0 * z[j];
        denom = lam + zr;
      }
      const double inv_den = 1.0 / denom;
      for (int r = 0; r < 7; r++) k[r] = Pz[r] * inv_den;
      const double e = y - yh;
      for (int j = 0; j < 7; j++) w[j] = w[j] + k[j] * e;
      if (sym) {
        for (int r = 0; r < 7; r++)
          for (int j = 0; j < 7; j++) P[r * 7 + j] = (P[r * 7 + j] - (Pz[r] * Pz[j]) * inv_den) * inv_lam;
      } else {
        double Pn[49];
        for (int r = 0; r < 7; r++)
          for (int j = 0; j < 7; j++) Pn[r * 7 + j] = (P[r * 7 + j] - k[r] * Pz[j]) * inv_lam;
        for (int r = 0; r < 7; r++)
          for (int j = 0; j < 7; j++) P[r * 7 + j] = 0.5 * (Pn[r * 7 + j] + Pn[j * 7 + r]);
      }
      bool fin = true;
      for (int j = 0; j < 7; j++) fin &= isfinite(w[j]);
      for (int j = 0; j < 7; j++) out[j] = w[j];
      for (int i = 0; i < 49; i++) out[7 + i] = P[i];
      out[56] = yh;
      out[57] = (double)(st | (fin ? 0 : 1));
      break;
    }
    default:
      out[0] = NAN;
  }
}

}  // namespace

extern "C" {

int intf_scalar(int32_t op, const uint64_t* args, int32_t n_args, double* out, int32_t n_out, void* stream) {
  INTF_RANGE("intf_scalar");
  if (!args || !out || n_args < 0 || n_args > 72 || n_out < 1 || n_out > 64 || op < 0 || op > INTF_SCALAR_RLS)
    return bad_input("intf_scalar: bad argument");
  static thread_local double* mapped = nullptr;  // per host thread: 64 doubles of mapped pinned memory
  static thread_local double* mapped_dev = nullptr;
  if (!mapped) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&mapped), 64 * sizeof(double), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped_dev), mapped, 0) != cudaSuccess) {
      mapped = nullptr;
      return launch_status("intf_scalar: mapped host buffer");
    }
  }
  ScalarArgs a;
  memset(&a, 0, sizeof(a));
  memcpy(a.u, args, sizeof(uint64_t) * n_args);
  cudaStream_t st = as_stream(stream);
  k_scalar<<<1, 32, 0, st>>>(op, a, mapped_dev);
  int rc = launch_status("k_scalar");
  if (rc) return rc;
  if (cudaStreamSynchronize(st) != cudaSuccess) return launch_status("intf_scalar: synchronize");
  memcpy(out, mapped, sizeof(double) * n_out);
  return INTF_OK;
}

int intf_noise_draws(uint64_t seed, double sigma, const int64_t* batch, const int64_t* seg, int64_t n, double* out,
                     void* stream) {
  INTF_RANGE("intf_noise_draws");
  if (!batch || !seg || !out || n < 0) return bad_input("intf_noise_draws: bad argument");
  if (n == 0) return INTF_OK;
  k_noise<<<ceil_div(n, 128), 128, 0, as_stream(stream)>>>(seed, sigma, batch, seg, (long long)n, out);
  return launch_status("k_noise");
}

int intf_slowdowns(const double* own, const double* colo, const double* beta, const double* noise, int64_t n,
                   double* out, void* stream) {
  INTF_RANGE("intf_slowdowns");
  if (!own || !colo || !beta || !out || n < 0) return bad_input("intf_slowdowns: bad argument");
  if (n == 0) return INTF_OK;
  k_slowdowns<<<ceil_div(n, 128), 128, 0, as_stream(stream)>>>(own, colo, beta[0], beta[1], beta[2], noise,
                                                               (long long)n, out);
  return launch_status("k_slowdowns");
}

int intf_rng_stream(const uint32_t* words, int32_t n_words, int64_t n, int32_t uniform, double* out, void* stream) {
  INTF_RANGE("intf_rng_stream");
  if (!words || !out || n_words < 1 || n_words > 8 || n < 0) return bad_input("intf_rng_stream: bad argument");
  k_normals<<<1, 32, 0, as_stream(stream)>>>(words, n_words, (long long)n, uniform, out);
  return launch_status("k_normals");
}


int intf_features_rows(const double* own, const int64_t* seg_off, const int32_t* nseg, const double* colo,
                       const double* measured, const double* profiled, int64_t n, const intf_predictor* preds,
                       int32_t n_pred, double* X, double* y, double* yhat, void* stream) {
  INTF_RANGE("intf_features_rows");
  if (!own || !seg_off || !nseg || !colo || n < 0 || n_pred < 0 || n_pred > kMaxPredRows || (n_pred && !preds))
    return bad_input("intf_features_rows: bad argument");
  if (y && (!measured || !profiled)) return bad_input("intf_features_rows: y needs measured and profiled");
  if (n == 0) return INTF_OK;
  PredRowsBlock P;
  memset(&P, 0, sizeof(P));
  for (int i = 0; i < n_pred; i++) P.p[i] = preds[i];
  k_features_rows<<<ceil_div(n, 128), 128, 0, as_stream(stream)>>>(own, seg_off, nseg, colo, measured, profiled,
                                                                   (long long)n, P, n_pred, X, y, yhat);
  return launch_status("k_features_rows");
}

int intf_predict_rows(const double* X, int64_t n, const double* w, double* out, void* stream) {
  INTF_RANGE("intf_predict_rows");
  if (!X || !w || !out || n < 0) return bad_input("intf_predict_rows: bad argument");
  if (n == 0) return INTF_OK;
  k_predict_rows<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(X, (long long)n, w, out);
  return launch_status("k_predict_rows");
}

int intf_quantiles(const double* values, int64_t n, const double* ps, int32_t nq, double* out, void* stream) {
  INTF_RANGE("intf_quantiles");
  if (!values || !ps || !out || n < 1 || nq < 1 || nq > kMaxQ) return bad_input("intf_quantiles: bad argument");
  k_quantiles<<<1, kSelThreads, 0, as_stream(stream)>>>(values, (long long)n, ps, nq, out);
  return launch_status("k_quantiles");
}

int intf_latency_report(const int32_t* group, const double* arrival, const double* completion, const uint8_t* met,
                        int64_t n, int32_t n_groups, double cutoff, int32_t* out_n, int32_t* out_met, double* out_p,
                        void* stream) {
  INTF_RANGE("intf_latency_report");
  if (!group || !arrival || !completion || !met || !out_n || !out_met || !out_p || n < 0 || n_groups < 1)
    return bad_input("intf_latency_report: bad argument");
  k_latency_report<<<n_groups, kSelThreads, 0, as_stream(stream)>>>(group, arrival, completion, met, (long long)n,
                                                                    cutoff, out_n, out_met, out_p);
  return launch_status("k_latency_report");
}

}  // extern "C"
