// predict.cu -- predictor-side kernels (sm_100a):
//   K5' candidate co-location sets: implicit enumeration, coarse + fine
//       predictions for many decisions (HBM-write bound)
//   K6  OLS normal-equation statistics (HBM-read bound) + 7x7 fp64 solve
//                                                   `predict.py:53-72,112-134`
//   K7  prequential SGD (thread per stream) / RLS (8 lanes per stream) `predict.py:75-205`
//   K8  EvalReport: MSE + nearest-rank relative-error quantiles
//                                                   `predict.py:176-205`
#include <math.h>

#include "capi_common.h"
#include "replay_core.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

using namespace intf;

namespace {

// ===================================================================== C2
// Candidate c = (own row o, multiset of k <= cap-1 peer rows).  Per own row
// the multisets are ranked size-major (k = 0, 1, ..) and in colex order
// within a size: multiset p1<=..<=pk <-> combination c_i = p_i + (i-1) of
// {0..E+k-2}, rank = sum_i C(c_i, i).
//
// Output layout (fp32), tiled so that every block of the streaming kernels
// writes ONE contiguous 16 KB tile (DRAM row locality: 6.2 vs 5.9 TB/s for the
// same bytes, tools/cand_stream_variants.cu v32 vs v3):
//   tile (dc, own, rc) = [kTileD decisions][2 kinds][kTileR multisets],
//   tiles ordered [dc = dec / kTileD][own][rc = r / kTileR],
// i.e. out[tile_off(dec, kind, own, r)], r < n_sets; ld = n_sets rounded up to
// kTileR (pad lanes written as 0), decisions padded to kTileD (the pad rows of
// the last tile are not written).  engine.CandidateScorer.view gives the
// logical [dec][kind][own][r] array.
constexpr int kMaxPeers = 7;  // cap <= 8

__host__ __device__ __forceinline__ long long binom(long long n, int k) {
  if (k < 0 || n < k) return 0;
  long long r = 1;
  for (int i = 1; i <= k; i++) r = r * (n - k + i) / i;
  return r;
}

long long n_multisets(int E, int cap) {
  long long sets = 0;
  for (int k = 0; k < cap; k++) sets += binom(E + k - 1, k);
  return sets;
}

constexpr int kCandThreads = 128;
constexpr int kOwnChunk = 4;
constexpr int kDecChunk = 32;
constexpr int kGroup = 4;  // multisets per thread (one float4 per output row)
constexpr int kTileR = 512;  // multisets per tile row (128 threads x kGroup)
constexpr int kTileD = 4;    // decisions per tile

__host__ __device__ __forceinline__ long long cand_ld(long long sets) { return (sets + kTileR - 1) / kTileR * kTileR; }
__host__ __device__ __forceinline__ long long cand_out_elems(int E, long long ld, int n_dec) {
  return (long long)(n_dec + kTileD - 1) / kTileD * kTileD * 2 * E * ld;
}
// element (dec, kind, own, r) of the tiled output
__device__ __forceinline__ long long tile_off(int d, int k, int o, long long r, int E, long long ld) {
  const long long RC = ld / kTileR;
  return ((((long long)(d / kTileD) * E + o) * RC + r / kTileR) * (2 * kTileD) + (d % kTileD) * 2 + k) * kTileR +
         r % kTileR;
}

// binomial table in shared memory: C[i][n] = binom(n, i), i <= kmax, n < nmax
struct BinomTab {
  const unsigned long long* c;
  int nmax;
  __device__ __forceinline__ unsigned long long operator()(int n, int i) const {
    return (n < i || n < 0) ? 0ull : c[i * nmax + n];
  }
};

template <int KMAX>
__device__ __forceinline__ int unrank_multiset(long long r, int E, int cap, const BinomTab& C, int* p) {
  int k = 0;
  for (; k < cap; k++) {
    const long long nk = (long long)C(E + k - 1, k);
    if (r < nk) break;
    r -= nk;
  }
#pragma unroll
  for (int i = KMAX; i >= 1; i--) {
    if (i > k) continue;
    int c;  // largest c with C(c, i) <= r
    if (i <= 3) {
      // closed-form estimate from C(c, i) ~ c^i / i!, then exact integer fix-up
      const double rr = (double)r;
      c = i == 1 ? (int)r : i == 2 ? (int)floor(0.5 * (1.0 + sqrt(1.0 + 8.0 * rr))) : (int)floor(cbrt(6.0 * rr)) + 1;
      c = c < i - 1 ? i - 1 : (c > E + k - 2 ? E + k - 2 : c);
      while (c > i - 1 && (long long)C(c, i) > r) c--;
      while (c < E + k - 2 && (long long)C(c + 1, i) <= r) c++;
    } else {
      int lo = i - 1, hi = E + k - 2;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((long long)C(mid, i) <= r) lo = mid;
        else hi = mid - 1;
      }
      c = lo;
    }
    r -= (long long)C(c, i);
    p[i - 1] = c - (i - 1);
  }
  return k;
}

// grid: x = groups of kGroup multisets, y = own-row chunks, z = decision chunks.
// Per multiset (fp64, amortised over kOwnChunk owns x kDecChunk decisions):
// colo snapshot with all peers ((0+p1)+p2).. (`simcore.py:126-131`), the
// departure history in (solo, row) order and its EWMA(alpha) prefixes
// (`colocation.py:54-63`).  Per prediction (fp32, within the 1e-5 budget):
// y = fma(w5, c2, fma(w4, c1, fma(w3, c0, bias))), bias = b + fp64 fma chain
// over the own features, one float4 {w3, w4, w5, bias} per (dec, kind, own)
// in shared memory.
// round to fp32 here (keeps the selects below on 32-bit registers)
__device__ __forceinline__ float to_f32(double v) {
  float r;
  asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(v));
  return r;
}

template <int KMAX>
__global__ void __launch_bounds__(kCandThreads, 2) k_candidates(const double* __restrict__ solo,
                                                                const double* __restrict__ thr, int E, int cap,
                                                                long long n_sets, long long ld, double alpha,
                                                                const double* __restrict__ coefs, int n_dec,
                                                                float* __restrict__ out) {
  extern __shared__ unsigned long long binom_smem[];
  __shared__ float4 cw[kDecChunk][2][kOwnChunk];
  __shared__ double own_solo[kOwnChunk];
  const int nmax = E + KMAX + 1;
  for (int t = threadIdx.x; t < (KMAX + 1) * nmax; t += blockDim.x) {
    const int i = t / nmax, n = t % nmax;
    binom_smem[t] = (unsigned long long)binom(n, i);
  }
  const int o0 = blockIdx.y * kOwnChunk, no = min(kOwnChunk, E - o0);
  const int d0 = blockIdx.z * kDecChunk, nd = min(kDecChunk, n_dec - d0);
  for (int t = threadIdx.x; t < kDecChunk * 2 * kOwnChunk; t += blockDim.x) {
    const int oi = t % kOwnChunk, kind = (t / kOwnChunk) & 1, d = t / (2 * kOwnChunk);
    if (oi < no && d < nd) {
      const double* w = coefs + ((d0 + d) * 2 + kind) * 7;
      const double* x = thr + 3 * (o0 + oi);
      const double bias = fma(w[2], x[2], fma(w[1], x[1], fma(w[0], x[0], 0.0))) + w[6];
      cw[d][kind][oi] = make_float4((float)w[3], (float)w[4], (float)w[5], (float)bias);
    }
  }
  if (threadIdx.x < no) own_solo[threadIdx.x] = solo[o0 + threadIdx.x];
  __syncthreads();
  const BinomTab C{binom_smem, nmax};
  const long long r0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kGroup;
  if (r0 >= ld) return;

  constexpr int KP = KMAX > 0 ? KMAX : 1;
  float c0[kGroup][3], ew[kGroup][KMAX + 1][3];
  unsigned jpack[kGroup];  // 3-bit departure counts, one per own in the chunk
  bool live[kGroup];
  const double om = 1.0 - alpha;
#pragma unroll
  for (int g = 0; g < kGroup; g++) {
    const long long r = r0 + g;
    int p[KP];
    live[g] = r < n_sets;
    const int k = live[g] ? unrank_multiset<KMAX>(r, E, cap, C, p) : 0;
    double th[KP][3], sp[KP];
#pragma unroll
    for (int q = 0; q < KMAX; q++) {
      const int row = q < k ? p[q] : 0;
      th[q][0] = thr[3 * row];
      th[q][1] = thr[3 * row + 1];
      th[q][2] = thr[3 * row + 2];
      sp[q] = q < k ? solo[row] : INFINITY;
    }
    // departure rank of each peer: order (solo, row); p is row-sorted
    int rk[KP];
#pragma unroll
    for (int q = 0; q < KMAX; q++) {
      int rq = 0;
#pragma unroll
      for (int j = 0; j < KMAX; j++)
        if (j != q && j < k && (sp[j] < sp[q] || (sp[j] == sp[q] && j < q))) rq++;
      rk[q] = rq;
    }
    // snapshot i = fresh sum, in row order, of the peers not yet departed
    // ((0+p1)+p2).. (`simcore.py:126-131`); EWMA prefixes (`colocation.py:61`)
    double e[3];
#pragma unroll
    for (int i = 0; i <= KMAX; i++) {
      double c[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < KMAX; q++)
        if (q < k && rk[q] >= i) {
          c[0] = c[0] + th[q][0];
          c[1] = c[1] + th[q][1];
          c[2] = c[2] + th[q][2];
        }
#pragma unroll
      for (int a = 0; a < 3; a++) {
        e[a] = i == 0 ? c[a] : alpha * c[a] + om * e[a];
        ew[g][i][a] = to_f32(e[a]);
        if (i == 0) c0[g][a] = ew[g][0][a];
      }
    }
    // peers that finish before each own row of the chunk (fp64 compare)
    unsigned jp = 0u;
#pragma unroll
    for (int oi = 0; oi < kOwnChunk; oi++) {
      const double so = own_solo[oi < no ? oi : 0];
      unsigned j = 0;
#pragma unroll
      for (int q = 0; q < KMAX; q++) j += (sp[q] < so) ? 1u : 0u;
      jp |= j << (3 * oi);
    }
    jpack[g] = jp;
  }
  const bool all_live = live[kGroup - 1];
  for (int oi = 0; oi < no; oi++) {
    float fe[kGroup][3];
#pragma unroll
    for (int g = 0; g < kGroup; g++) {
      const unsigned j = (jpack[g] >> (3 * oi)) & 7u;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        float v = ew[g][0][a];
#pragma unroll
        for (int i = 1; i <= KMAX; i++) v = (i == (int)j) ? ew[g][i][a] : v;
        fe[g][a] = v;
      }
    }
    // dead pad lanes (r >= n_sets) compute from zeroed features; zero them at store
#pragma unroll 4
    for (int d = 0; d < nd; d++) {
      float* rowc = out + tile_off(d0 + d, 0, o0 + oi, r0, E, ld);
      const long long kstride = kTileR;  // the fine row follows the coarse row in the tile
      const float4 a = cw[d][0][oi];
      const float4 b = cw[d][1][oi];
      float yc[kGroup], yf[kGroup];
#pragma unroll
      for (int g = 0; g < kGroup; g++) {
        yc[g] = fmaf(a.z, c0[g][2], fmaf(a.y, c0[g][1], fmaf(a.x, c0[g][0], a.w)));
        yf[g] = fmaf(b.z, fe[g][2], fmaf(b.y, fe[g][1], fmaf(b.x, fe[g][0], b.w)));
      }
      if (all_live) {
        __stcs(reinterpret_cast<float4*>(rowc), make_float4(yc[0], yc[1], yc[2], yc[3]));
        __stcs(reinterpret_cast<float4*>(rowc + kstride), make_float4(yf[0], yf[1], yf[2], yf[3]));
      } else {
        __stcs(reinterpret_cast<float4*>(rowc), make_float4(live[0] ? yc[0] : 0.f, live[1] ? yc[1] : 0.f,
                                                            live[2] ? yc[2] : 0.f, live[3] ? yc[3] : 0.f));
        __stcs(reinterpret_cast<float4*>(rowc + kstride), make_float4(live[0] ? yf[0] : 0.f, live[1] ? yf[1] : 0.f,
                                                                      live[2] ? yf[2] : 0.f, live[3] ? yf[3] : 0.f));
      }
    }
  }
}

// ---- two-phase form for tables whose per-(multiset, own) feature table
// fits comfortably in L2 (the 48-row bundled table: 12 MB).
// Phase 1 (k_cand_prep): one thread per multiset decodes it once and writes
//   C0[c][r]          static colo snapshot (fp32)
//   FE[(o*3 + c)][r]  EWMA features seen by own row o (the prefix selected by
//                     how many peers finish before o), fp32
// Phase 2 (k_cand_stream): pure streaming -- per thread 4 multisets x 1 own x
// kStreamDec decisions: 3 FFMA per prediction, 16-byte streaming stores.
// own rows per prep thread (grid.y splits the table): 12 for the standalone
// k_cand_prep (shortest launch), 48 inside the fused k_cand_step, where the
// 163 prep blocks run beside the stream blocks and fewer, longer blocks
// disturb them least (B200, C2 shape: 43.2 us/step at 48 vs 44.1 at 12).
constexpr int kPrepOwn = 12;
constexpr int kStepPrepOwn = 48;

template <int KMAX>
__device__ __forceinline__ void cand_prep_body(int bx, int by, const double* __restrict__ solo,
                                               const double* __restrict__ thr, int E, int cap, long long n_sets,
                                               long long ld, double alpha, float* __restrict__ C0,
                                               float* __restrict__ FE, int prep_own) {
  extern __shared__ unsigned long long binom_smem[];
  const int nmax = E + KMAX + 1;
  for (int t = threadIdx.x; t < (KMAX + 1) * nmax; t += blockDim.x) {
    const int i = t / nmax, n = t % nmax;
    binom_smem[t] = (unsigned long long)binom(n, i);
  }
  __syncthreads();
  const BinomTab C{binom_smem, nmax};
  const long long r = (long long)bx * blockDim.x + threadIdx.x;
  if (r >= ld) return;
  constexpr int KP = KMAX > 0 ? KMAX : 1;
  const bool live = r < n_sets;
  int p[KP];
  const int k = live ? unrank_multiset<KMAX>(r, E, cap, C, p) : 0;
  double th[KP][3], sp[KP];
#pragma unroll
  for (int q = 0; q < KMAX; q++) {
    const int row = q < k ? p[q] : 0;
    th[q][0] = thr[3 * row];
    th[q][1] = thr[3 * row + 1];
    th[q][2] = thr[3 * row + 2];
    sp[q] = q < k ? solo[row] : INFINITY;
  }
  int rk[KP];
#pragma unroll
  for (int q = 0; q < KMAX; q++) {
    int rq = 0;
#pragma unroll
    for (int j = 0; j < KMAX; j++)
      if (j != q && j < k && (sp[j] < sp[q] || (sp[j] == sp[q] && j < q))) rq++;
    rk[q] = rq;
  }
  float ew[KMAX + 1][3];
  double e[3];
  const double om = 1.0 - alpha;
  const int o_begin = by * prep_own, o_end = min(E, o_begin + prep_own);
#pragma unroll
  for (int i = 0; i <= KMAX; i++) {
    double c[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < KMAX; q++)
      if (q < k && rk[q] >= i) {
        c[0] = c[0] + th[q][0];
        c[1] = c[1] + th[q][1];
        c[2] = c[2] + th[q][2];
      }
#pragma unroll
    for (int a = 0; a < 3; a++) {
      e[a] = i == 0 ? c[a] : alpha * c[a] + om * e[a];
      ew[i][a] = live ? to_f32(e[a]) : 0.0f;
    }
  }
  if (by == 0) {
#pragma unroll
    for (int a = 0; a < 3; a++) C0[a * ld + r] = ew[0][a];
  }
  for (int o = o_begin; o < o_end; o++) {
    const double so = solo[o];
    int j = 0;
#pragma unroll
    for (int q = 0; q < KMAX; q++) j += (sp[q] < so) ? 1 : 0;  // peers that finish first
#pragma unroll
    for (int a = 0; a < 3; a++) {
      float v = ew[0][a];
#pragma unroll
      for (int i = 1; i <= KMAX; i++) v = (i == j) ? ew[i][a] : v;
      FE[((long long)o * 3 + a) * ld + r] = v;
    }
  }
}

constexpr int kStreamThreads = 128;
// decisions per block: 4 (x 2 kinds = 8 float4 stores per thread).  Short
// blocks stream best -- measured on B200 for the C2 shape (tools/
// cand_stream_variants.cu): 32 per block 5.09 TB/s, 16: 5.24, 8: 5.56,
// 4: 5.89, 2: 5.20; a one-float4-per-thread fill reaches 6.50.
constexpr int kStreamDec = 4;
static_assert(kStreamDec == kTileD && kStreamThreads * kGroup == kTileR, "a stream block writes exactly one tile");
static_assert(kCandThreads * kGroup == kTileR, "k_candidates blocks cover one tile column");

// grid: x = groups of 4 multisets, y = own row, z = decision chunks.  The
// thread's feature loads (L2-resident C0/FE) are issued before the block
// builds its coefficient slab, so their latency overlaps that setup.
// kBest: instead of storing every prediction, reduce them per (decision,
// kind, own) to the best candidate -- the minimum predicted interference
// ratio, ties to the lowest multiset rank -- as one 64-bit key
// (orderable(fp32 value) << 32 | rank) folded into best[] by atomicMin:
// warp minima by redux.sync on the value key and then on the rank among the
// lanes holding it, block minima through shared memory, one atomic per
// (decision, kind) per block.
__device__ __forceinline__ unsigned f32_key(float v) {
  const unsigned u = __float_as_uint(v);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}

constexpr int kBestSpan = 4;  // groups of 4 multisets per thread in the best-candidate reduction

template <bool kBest>
__device__ __forceinline__ void cand_stream_body(int bx, int by, int bz, const double* __restrict__ thr, int E,
                                                 long long ld, long long n_sets, const double* __restrict__ coefs,
                                                 int n_dec, const float* __restrict__ C0,
                                                 const float* __restrict__ FE, float* __restrict__ out,
                                                 unsigned long long* __restrict__ best = nullptr) {
  __shared__ float4 cw[kStreamDec][2];
  const int o = by;
  const int d0 = bz * kStreamDec, nd = min(kStreamDec, n_dec - d0);
  if constexpr (kBest) {
    // kBestSpan groups of 4 multisets per thread (strided by the block, so
    // loads stay coalesced): the warp / block reductions amortise over 16
    // multisets instead of 4; nothing is written per candidate
    for (int t = threadIdx.x; t < 2 * nd; t += blockDim.x) {
      const int d = t >> 1, kind = t & 1;
      const double* w = coefs + ((d0 + d) * 2 + kind) * 7;
      const double* x = thr + 3 * o;
      const double bias = fma(w[2], x[2], fma(w[1], x[1], fma(w[0], x[0], 0.0))) + w[6];
      cw[d][kind] = make_float4((float)w[3], (float)w[4], (float)w[5], (float)bias);
    }
    __syncthreads();
    __shared__ unsigned red_v[kStreamThreads / 32][kStreamDec][2], red_i[kStreamThreads / 32][kStreamDec][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per thread: the running minimum as a float and its rank (a key only for
    // the warp reduction: one FSETP + two selects per prediction)
    float bc[kStreamDec], bf[kStreamDec];
    unsigned ic[kStreamDec], jf[kStreamDec];
#pragma unroll
    for (int d = 0; d < kStreamDec; d++) bc[d] = bf[d] = INFINITY, ic[d] = jf[d] = 0xffffffffu;
#pragma unroll
    for (int c = 0; c < kBestSpan; c++) {
      const long long r0 = (((long long)bx * kBestSpan + c) * blockDim.x + threadIdx.x) * 4;
      const long long nl = r0 < ld ? n_sets - r0 : 0;  // valid multisets of this group (<= 0: none)
      const long long rr = r0 < ld ? r0 : 0;
      const float4 cx = __ldg(reinterpret_cast<const float4*>(C0 + rr));
      const float4 cy = __ldg(reinterpret_cast<const float4*>(C0 + ld + rr));
      const float4 cz = __ldg(reinterpret_cast<const float4*>(C0 + 2 * ld + rr));
      const float4 fx = __ldg(reinterpret_cast<const float4*>(FE + ((long long)o * 3 + 0) * ld + rr));
      const float4 fy = __ldg(reinterpret_cast<const float4*>(FE + ((long long)o * 3 + 1) * ld + rr));
      const float4 fz = __ldg(reinterpret_cast<const float4*>(FE + ((long long)o * 3 + 2) * ld + rr));
#pragma unroll
      for (int d = 0; d < kStreamDec; d++) {
        if (d >= nd) break;
        const float4 a = cw[d][0], b = cw[d][1];
        const float yc[4] = {fmaf(a.z, cz.x, fmaf(a.y, cy.x, fmaf(a.x, cx.x, a.w))),
                             fmaf(a.z, cz.y, fmaf(a.y, cy.y, fmaf(a.x, cx.y, a.w))),
                             fmaf(a.z, cz.z, fmaf(a.y, cy.z, fmaf(a.x, cx.z, a.w))),
                             fmaf(a.z, cz.w, fmaf(a.y, cy.w, fmaf(a.x, cx.w, a.w)))};
        const float yf[4] = {fmaf(b.z, fz.x, fmaf(b.y, fy.x, fmaf(b.x, fx.x, b.w))),
                             fmaf(b.z, fz.y, fmaf(b.y, fy.y, fmaf(b.x, fx.y, b.w))),
                             fmaf(b.z, fz.z, fmaf(b.y, fy.z, fmaf(b.x, fx.z, b.w))),
                             fmaf(b.z, fz.w, fmaf(b.y, fy.w, fmaf(b.x, fx.w, b.w)))};
#pragma unroll
        for (int i = 0; i < 4; i++) {
          if (i < nl) {  // groups in ascending rank: strict < keeps the lowest rank on ties
            if (yc[i] < bc[d]) bc[d] = yc[i], ic[d] = (unsigned)(r0 + i);
            if (yf[i] < bf[d]) bf[d] = yf[i], jf[d] = (unsigned)(r0 + i);
          }
        }
      }
    }
    for (int d = 0; d < nd; d++) {
      const unsigned vc = ic[d] == 0xffffffffu ? 0xffffffffu : f32_key(bc[d]);
      const unsigned vf = jf[d] == 0xffffffffu ? 0xffffffffu : f32_key(bf[d]);
      const unsigned wc = __reduce_min_sync(0xffffffffu, vc), wf = __reduce_min_sync(0xffffffffu, vf);
      const unsigned xc = __reduce_min_sync(0xffffffffu, vc == wc ? ic[d] : 0xffffffffu);
      const unsigned xf = __reduce_min_sync(0xffffffffu, vf == wf ? jf[d] : 0xffffffffu);
      if (lane == 0) {
        red_v[warp][d][0] = wc, red_i[warp][d][0] = xc;
        red_v[warp][d][1] = wf, red_i[warp][d][1] = xf;
      }
    }
    __syncthreads();
    if (threadIdx.x < 2 * nd) {
      const int d = threadIdx.x >> 1, kind = threadIdx.x & 1;
      unsigned long long key = ~0ull;
#pragma unroll
      for (int w = 0; w < kStreamThreads / 32; w++) {
        const unsigned long long k2 = ((unsigned long long)red_v[w][d][kind] << 32) | red_i[w][d][kind];
        key = k2 < key ? k2 : key;
      }
      if (key != ~0ull) atomicMin(best + ((long long)(d0 + d) * 2 + kind) * E + o, key);
    }
    return;
  }
  const long long r0 = ((long long)bx * blockDim.x + threadIdx.x) * 4;
  const bool inb = r0 < ld;
  const long long rr = inb ? r0 : 0;
  const float4 cx = __ldg(reinterpret_cast<const float4*>(C0 + rr));
  const float4 cy = __ldg(reinterpret_cast<const float4*>(C0 + ld + rr));
  const float4 cz = __ldg(reinterpret_cast<const float4*>(C0 + 2 * ld + rr));
  const float4 fx = __ldg(reinterpret_cast<const float4*>(FE + ((long long)o * 3 + 0) * ld + rr));
  const float4 fy = __ldg(reinterpret_cast<const float4*>(FE + ((long long)o * 3 + 1) * ld + rr));
  const float4 fz = __ldg(reinterpret_cast<const float4*>(FE + ((long long)o * 3 + 2) * ld + rr));
  for (int t = threadIdx.x; t < 2 * nd; t += blockDim.x) {
    const int d = t >> 1, kind = t & 1;
    const double* w = coefs + ((d0 + d) * 2 + kind) * 7;
    const double* x = thr + 3 * o;
    const double bias = fma(w[2], x[2], fma(w[1], x[1], fma(w[0], x[0], 0.0))) + w[6];
    cw[d][kind] = make_float4((float)w[3], (float)w[4], (float)w[5], (float)bias);
  }
  __syncthreads();
  if (!inb) return;
  const long long nl = n_sets - r0;  // < 4 only in the last group: pad lanes are written as 0
  // this block's tile: (dc = bz, own = o, rc = bx), rows (dec % 4, kind) of kTileR floats
  float* row = out + tile_off(d0, 0, o, r0, E, ld);
#pragma unroll 4
  for (int d = 0; d < nd; d++) {
    const float4 a = cw[d][0], b = cw[d][1];
    float4 yc, yf;
    yc.x = fmaf(a.z, cz.x, fmaf(a.y, cy.x, fmaf(a.x, cx.x, a.w)));
    yc.y = fmaf(a.z, cz.y, fmaf(a.y, cy.y, fmaf(a.x, cx.y, a.w)));
    yc.z = fmaf(a.z, cz.z, fmaf(a.y, cy.z, fmaf(a.x, cx.z, a.w)));
    yc.w = fmaf(a.z, cz.w, fmaf(a.y, cy.w, fmaf(a.x, cx.w, a.w)));
    yf.x = fmaf(b.z, fz.x, fmaf(b.y, fy.x, fmaf(b.x, fx.x, b.w)));
    yf.y = fmaf(b.z, fz.y, fmaf(b.y, fy.y, fmaf(b.x, fx.y, b.w)));
    yf.z = fmaf(b.z, fz.z, fmaf(b.y, fy.z, fmaf(b.x, fx.z, b.w)));
    yf.w = fmaf(b.z, fz.w, fmaf(b.y, fy.w, fmaf(b.x, fx.w, b.w)));
    if (nl < 4) {
      yc = make_float4(nl > 0 ? yc.x : 0.f, nl > 1 ? yc.y : 0.f, nl > 2 ? yc.z : 0.f, 0.f);
      yf = make_float4(nl > 0 ? yf.x : 0.f, nl > 1 ? yf.y : 0.f, nl > 2 ? yf.z : 0.f, 0.f);
    }
    __stcs(reinterpret_cast<float4*>(row), yc);
    __stcs(reinterpret_cast<float4*>(row + kTileR), yf);
    row += 2 * kTileR;
  }
}

template <int KMAX>
__global__ void __launch_bounds__(128) k_cand_prep(const double* __restrict__ solo, const double* __restrict__ thr,
                                                   int E, int cap, long long n_sets, long long ld, double alpha,
                                                   float* __restrict__ C0, float* __restrict__ FE, int prep_own) {
  cand_prep_body<KMAX>(blockIdx.x, blockIdx.y, solo, thr, E, cap, n_sets, ld, alpha, C0, FE, prep_own);
}

__global__ void __launch_bounds__(kStreamThreads, 8) k_cand_stream(const double* __restrict__ thr, int E, long long ld,
                                                                   long long n_sets,
                                                                   const double* __restrict__ coefs, int n_dec,
                                                                   const float* __restrict__ C0,
                                                                   const float* __restrict__ FE,
                                                                   float* __restrict__ out) {
  cand_stream_body<false>(blockIdx.x, blockIdx.y, blockIdx.z, thr, E, ld, n_sets, coefs, n_dec, C0, FE, out);
}

// One pipelined step in ONE launch: the forward of every candidate from the
// features in ws_cur (stream blocks) + the feature build for the next step
// into ws_next (prep blocks), horizontally fused so the issue-bound prep work
// fills the HBM-bound stream kernel's idle issue slots and no cross-stream
// synchronisation or second launch sits between steps.  1-D grid: the first
// n_prep blocks are prep blocks (dispatched first, they run beside the
// stream blocks instead of after them).
// kBest: the stream blocks reduce to best[] (see cand_stream_body) and the
// prep blocks also reset best_next[0, n_best) for the next step.
template <int KMAX, bool kBest = false>
__global__ void __launch_bounds__(kStreamThreads, 8) k_cand_step(
    const double* __restrict__ solo, const double* __restrict__ thr, int E, int cap, long long n_sets, long long ld,
    double alpha, const double* __restrict__ coefs, int n_dec, const float* __restrict__ ws_cur,
    float* __restrict__ ws_next, float* __restrict__ out, int prep_x, int prep_y, int prep_own, int stream_x,
    unsigned long long* __restrict__ best = nullptr, unsigned long long* __restrict__ best_next = nullptr,
    long long n_best = 0) {
  // programmatic dependent launch: let the next step's grid be scheduled as
  // soon as every CTA of this one is running, and wait for the previous
  // step's grid (its prep blocks wrote ws_cur; its stream blocks read
  // ws_next) before touching memory.  Both are no-ops without PDL.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_prep = ws_next ? prep_x * prep_y : 0;
  int b = blockIdx.x;
  if (b < n_prep) {
    cand_prep_body<KMAX>(b % prep_x, b / prep_x, solo, thr, E, cap, n_sets, ld, alpha, ws_next, ws_next + 3 * ld,
                         prep_own);
    if constexpr (kBest) {
      if (best_next)
        for (long long i = (long long)b * blockDim.x + threadIdx.x; i < n_best; i += (long long)n_prep * blockDim.x)
          best_next[i] = ~0ull;
    }
    return;
  }
  b -= n_prep;
  const int bx = b % stream_x, rest = b / stream_x;
  cand_stream_body<kBest>(bx, rest % E, rest / E, thr, E, ld, n_sets, coefs, n_dec, ws_cur, ws_cur + 3 * ld, out, best);
}

// The host-buffer best-candidate call in ONE launch (intf_best_candidates_host_
// pipelined with a pinned result buffer): the decisions' coefficients arrive
// as a kernel parameter (no host->device copy), and the last stream block to
// finish (a completion counter) copies the reduced keys straight into the
// caller's pinned buffer over the bus and re-arms them (~0) for the next
// call (no device->host copy, no memset).  The next call's blocks wait for
// this grid (griddepcontrol.wait) before touching memory.
constexpr int kHostDecMax = 32;  // decisions whose coefficients fit the 4 KB parameter space
struct CandCoefs {
  double c[kHostDecMax * 2 * 7];
};
template <int KMAX>
__global__ void __launch_bounds__(kStreamThreads, 8) k_cand_step_host(
    const double* __restrict__ solo, const double* __restrict__ thr, int E, int cap, long long n_sets, long long ld,
    double alpha, const __grid_constant__ CandCoefs cp, int n_dec, const float* __restrict__ ws_cur,
    float* __restrict__ ws_next, int prep_x, int prep_y, int prep_own, int stream_x,
    unsigned long long* __restrict__ best, long long n_best, unsigned* __restrict__ done, int n_stream_blocks,
    unsigned long long* __restrict__ host_best, volatile unsigned long long* flag, unsigned long long seq) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_prep = ws_next ? prep_x * prep_y : 0;
  int b = blockIdx.x;
  if (b < n_prep) {
    cand_prep_body<KMAX>(b % prep_x, b / prep_x, solo, thr, E, cap, n_sets, ld, alpha, ws_next, ws_next + 3 * ld,
                         prep_own);
    return;
  }
  b -= n_prep;
  const int bx = b % stream_x, rest = b / stream_x;
  cand_stream_body<true>(bx, rest % E, rest / E, thr, E, ld, n_sets, cp.c, n_dec, ws_cur, ws_cur + 3 * ld, nullptr,
                         best);
  __shared__ bool last;
  __threadfence();  // this block's atomicMin results before its count
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == (unsigned)n_stream_blocks - 1u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const ulonglong2* src = reinterpret_cast<const ulonglong2*>(best);
  ulonglong2* dst = reinterpret_cast<ulonglong2*>(host_best);
  for (long long i = threadIdx.x; i < n_best / 2; i += blockDim.x) {
    dst[i] = __ldcg(src + i);
    reinterpret_cast<ulonglong2*>(best)[i] = make_ulonglong2(~0ull, ~0ull);
  }
  if ((n_best & 1) && threadIdx.x == 0) {
    host_best[n_best - 1] = __ldcg(best + n_best - 1);
    best[n_best - 1] = ~0ull;
  }
  if (threadIdx.x == 0) *done = 0u;
  if (flag) {  // the waiting host thread's signal: every key store of the block before it
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *flag = seq;
  }
}

// ---- real scheduling decisions ("the per-decision candidate
// set from C5 replays").  Decision = the dispatch of batch b of a replayed
// scenario; its running set = the batches it co-runs with right after the
// dispatch (dispatched before b -- FIFO, batch-id order -- and completing
// strictly after b's start: a batch completing at that very instant leaves
// within the same timestamp, `simcore.py:56-64`).  The set is written as its
// multiset rank in the candidate enumeration of cap_enum (size-major, colex),
// so the candidates of a decision are column r of the enumeration: every own
// row against that running set.  Thread per batch, block per scenario.
__global__ void k_dispatch_sets(const intf_scenario* __restrict__ scen, int n_scen,
                                const intf_model* __restrict__ models, intf_replay_buffers B, int E, int cap_enum,
                                int32_t* __restrict__ dec_rank, int32_t* __restrict__ dec_own) {
  for (int s = blockIdx.x; s < n_scen; s += gridDim.x) {
    const intf_scenario& S = scen[s];
    const long long ro = S.req_off;
    const int nb = B.n_batches[s];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const double tb = B.b_start[ro + b];
      const int nrun = B.b_running ? B.b_running[ro + b] : cap_enum;
      int peers[kMaxPeers];
      int k = 0;
      // the dispatch trace bounds the scan: nrun - 1 batches were running at the dispatch
      for (int c = b - 1; c >= 0 && k < nrun - 1 && k < cap_enum - 1; c--)
        if (B.b_completion[ro + c] > tb)
          peers[k++] = models[S.model_off + B.b_model[ro + c]].entry_base + B.b_size[ro + c] - 1;
      for (int i = 1; i < k; i++)  // ascending entries
        for (int j = i; j > 0 && peers[j - 1] > peers[j]; j--) {
          const int t = peers[j];
          peers[j] = peers[j - 1];
          peers[j - 1] = t;
        }
      long long r = 0;
      for (int j = 0; j < k; j++) r += binom(E + j - 1, j);
      for (int i = 0; i < k; i++) r += binom(peers[i] + i, i + 1);
      dec_rank[ro + b] = (int32_t)r;
      dec_own[ro + b] = models[S.model_off + B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1;
    }
  }
}

// warp per decision: every own row scored against the decision's running set
// (column r of the enumeration's features, the same fp32 arithmetic as
// cand_stream_body, so a prediction equals the enumeration's), then the best
// own row per predictor kind -- (orderable value << 32 | own) -- and the
// prediction for the batch FIFO actually dispatched.  n decisions at
// dec_rank[i] (< 0: none).
__global__ void __launch_bounds__(128) k_score_decisions(const double* __restrict__ thr, int E, long long ld,
                                                         const double* __restrict__ coefs,
                                                         const float* __restrict__ C0,
                                                         const float* __restrict__ FE,
                                                         const int32_t* __restrict__ dec_rank,
                                                         const int32_t* __restrict__ dec_own, long long n,
                                                         unsigned long long* __restrict__ best,
                                                         float* __restrict__ chosen,
                                                         const float* __restrict__ FT = nullptr) {
  __shared__ float4 cw[2][64];  // per own row: coarse / fine (w3, w4, w5, bias)
  for (int t = threadIdx.x; t < 2 * E; t += blockDim.x) {
    const int kind = t / E, o = t % E;
    const double* w = coefs + kind * 7;
    const double* x = thr + 3 * o;
    const double bias = fma(w[2], x[2], fma(w[1], x[1], fma(w[0], x[0], 0.0))) + w[6];
    cw[kind][o] = make_float4((float)w[3], (float)w[4], (float)w[5], (float)bias);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long n_warps = (long long)gridDim.x * (blockDim.x >> 5);
  // warps stride over 32-slot groups (the block's coefficient table is built
  // once): the group's ranks load coalesced, empty slots (no batch) are
  // marked in one store each, and the warp scores the group's decisions one
  // after the other
  for (long long base = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n;
       base += n_warps * 32) {
  const long long slot = base + lane;
  const int my_r = slot < n ? dec_rank[slot] : -1;
  const int my_own = slot < n ? dec_own[slot] : 0;
  if (slot < n && my_r < 0) {
    best[2 * slot] = best[2 * slot + 1] = ~0ull;
    chosen[2 * slot] = chosen[2 * slot + 1] = NAN;
  }
  for (unsigned todo = __ballot_sync(0xffffffffu, my_r >= 0); todo; todo &= todo - 1) {
  const int j = __ffs(todo) - 1;
  const long long i = base + j;
  const int r = __shfl_sync(0xffffffffu, my_r, j);
  const int own_b = __shfl_sync(0xffffffffu, my_own, j);
  const float cx = C0[r], cy = C0[ld + r], cz = C0[2 * ld + r];
  unsigned vc = 0xffffffffu, vf = 0xffffffffu, oc = 0xffffffffu, of = 0xffffffffu;
  for (int o = lane; o < E; o += 32) {
    const float4 a = cw[0][o], b = cw[1][o];
    float fx, fy, fz;
    if (FT) {  // decision-major copy: the 48 x 3 features of column r are contiguous
      const float* f = FT + ((long long)r * E + o) * 3;
      fx = f[0], fy = f[1], fz = f[2];
    } else {
      fx = FE[((long long)o * 3 + 0) * ld + r], fy = FE[((long long)o * 3 + 1) * ld + r],
      fz = FE[((long long)o * 3 + 2) * ld + r];
    }
    const float yc = fmaf(a.z, cz, fmaf(a.y, cy, fmaf(a.x, cx, a.w)));
    const float yf = fmaf(b.z, fz, fmaf(b.y, fy, fmaf(b.x, fx, b.w)));
    const unsigned kc = f32_key(yc), kf = f32_key(yf);
    if (kc < vc) vc = kc, oc = (unsigned)o;  // ascending own: strict < keeps the lowest on ties
    if (kf < vf) vf = kf, of = (unsigned)o;
    if (o == own_b) chosen[2 * i] = yc, chosen[2 * i + 1] = yf;
  }
#ifdef INTF_DECISION_REDUX
  const unsigned wc = __reduce_min_sync(0xffffffffu, vc), wf = __reduce_min_sync(0xffffffffu, vf);
  const unsigned xc = __reduce_min_sync(0xffffffffu, vc == wc ? oc : 0xffffffffu);
  const unsigned xf = __reduce_min_sync(0xffffffffu, vf == wf ? of : 0xffffffffu);
  const unsigned long long kc = ((unsigned long long)wc << 32) | xc, kf = ((unsigned long long)wf << 32) | xf;
#else
  // packed (value << 32 | own) keys: one 64-bit butterfly min per kind gives value and lowest own at once
  unsigned long long kc = ((unsigned long long)vc << 32) | oc, kf = ((unsigned long long)vf << 32) | of;
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) {
    const unsigned long long pc = __shfl_xor_sync(0xffffffffu, kc, o2), pf = __shfl_xor_sync(0xffffffffu, kf, o2);
    kc = pc < kc ? pc : kc;
    kf = pf < kf ? pf : kf;
  }
#endif
  if (lane == 0) {
    best[2 * i] = kc;
    best[2 * i + 1] = kf;
  }
  }
  }
}

// The same scores with a LANE per decision (decision-major features FT):
// each lane walks the 48 own rows of its decision's column, the coefficient
// rows are shared-memory broadcasts, and the features are the lane's own
// contiguous 576 B -- no shuffles, no per-decision reductions.  The same
// fp32 arithmetic per (rank, own) as cand_stream_body, the lowest own row on
// ties (ascending, strict <), so the results equal k_score_decisions'.
__global__ void __launch_bounds__(128) k_score_decisions_lane(const double* __restrict__ thr, int E, long long ld,
                                                              const double* __restrict__ coefs,
                                                              const float* __restrict__ C0,
                                                              const float* __restrict__ FT,
                                                              const int32_t* __restrict__ dec_rank,
                                                              const int32_t* __restrict__ dec_own, long long n,
                                                              unsigned long long* __restrict__ best,
                                                              float* __restrict__ chosen) {
  __shared__ float4 cw[2][64];  // per own row: coarse / fine (w3, w4, w5, bias)
  for (int t = threadIdx.x; t < 2 * E; t += blockDim.x) {
    const int kind = t / E, o = t % E;
    const double* w = coefs + kind * 7;
    const double* x = thr + 3 * o;
    const double bias = fma(w[2], x[2], fma(w[1], x[1], fma(w[0], x[0], 0.0))) + w[6];
    cw[kind][o] = make_float4((float)w[3], (float)w[4], (float)w[5], (float)bias);
  }
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = dec_rank[i];
    if (r < 0) {
      best[2 * i] = best[2 * i + 1] = ~0ull;
      chosen[2 * i] = chosen[2 * i + 1] = NAN;
      continue;
    }
    const int own_b = dec_own[i];
    const float cx = C0[r], cy = C0[ld + r], cz = C0[2 * ld + r];
    const float* f = FT + (long long)r * E * 3;
    unsigned vc = 0xffffffffu, vf = 0xffffffffu, oc = 0xffffffffu, of = 0xffffffffu;
    float yc_b = NAN, yf_b = NAN;
    auto own_row = [&](int o, float fx, float fy, float fz) {
      const float4 a = cw[0][o], b = cw[1][o];
      const float yc = fmaf(a.z, cz, fmaf(a.y, cy, fmaf(a.x, cx, a.w)));
      const float yf = fmaf(b.z, fz, fmaf(b.y, fy, fmaf(b.x, fx, b.w)));
      const unsigned kc = f32_key(yc), kf = f32_key(yf);
      if (kc < vc) vc = kc, oc = (unsigned)o;
      if (kf < vf) vf = kf, of = (unsigned)o;
      if (o == own_b) yc_b = yc, yf_b = yf;
    };
    int o = 0;
    if ((((unsigned long long)f) & 15) == 0) {  // 4 own rows = 12 floats = 3 aligned float4 loads
      for (; o + 4 <= E; o += 4) {
        const float4 p0 = *reinterpret_cast<const float4*>(f + 3 * o);
        const float4 p1 = *reinterpret_cast<const float4*>(f + 3 * o + 4);
        const float4 p2 = *reinterpret_cast<const float4*>(f + 3 * o + 8);
        own_row(o, p0.x, p0.y, p0.z);
        own_row(o + 1, p0.w, p1.x, p1.y);
        own_row(o + 2, p1.z, p1.w, p2.x);
        own_row(o + 3, p2.y, p2.z, p2.w);
      }
    }
    for (; o < E; o++) own_row(o, f[3 * o], f[3 * o + 1], f[3 * o + 2]);
    best[2 * i] = ((unsigned long long)vc << 32) | oc;
    best[2 * i + 1] = ((unsigned long long)vf << 32) | of;
    chosen[2 * i] = yc_b;
    chosen[2 * i + 1] = yf_b;
  }
}

// FT[r][own][3] = FE[own][a][r]: the EWMA candidate features in
// decision-major order (one transpose per table / cap / alpha) so a decision
// reads its column's 48 x 3 features contiguously instead of 144 rows apart
__global__ void k_decision_transpose(const float* __restrict__ FE, int E, long long ld, long long n_sets,
                                     float* __restrict__ FT) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // (r, own, a) in output order
  if (i >= n_sets * E * 3) return;
  const int a = (int)(i % 3);
  const long long t = i / 3;
  const int o = (int)(t % E);
  const long long r = t / E;
  FT[i] = FE[((long long)o * 3 + a) * ld + r];
}

// ===================================================================== K6
constexpr int kOlsThreads = 256;
constexpr int kOlsBlocks = 296;  // one wave: 2 x 148 SMs at 128 registers x 256 threads
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
  // 16-byte loads, four rows in flight per thread (X rows are 48 B: 16-byte
  // aligned); the accumulation order per thread is unchanged (row order)
#pragma unroll 4
  for (long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (long long)gridDim.x * blockDim.x) {
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

// cyclic Jacobi eigenvalues of a symmetric 7x7 (fp64), for the rank test.
// Fully unrolled so the matrix lives in registers (no local memory).
__device__ __forceinline__ void jacobi_eigs(const double* G, double* ev) {
  double a[7][7];
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = 0; j < 7; j++) a[i][j] = G[i * 7 + j];
  double fro = 0.0;  // ||G||_F^2: stop once the off-diagonal mass is below (eps ||G||_F)^2
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = 0; j < 7; j++) fro += a[i][j] * a[i][j];
  const double stop = fro * 1.2e-34;
  for (int sweep = 0; sweep < 30; sweep++) {
    double off = 0.0;
#pragma unroll
    for (int i = 0; i < 7; i++)
#pragma unroll
      for (int j = i + 1; j < 7; j++) off += a[i][j] * a[i][j];
    if (off <= stop) break;
#pragma unroll
    for (int p = 0; p < 7; p++)
#pragma unroll
      for (int q = p + 1; q < 7; q++) {
        const double apq = a[p][q];
        if (apq != 0.0) {
          const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
          for (int k = 0; k < 7; k++) {
            const double akp = a[k][p], akq = a[k][q];
            a[k][p] = c * akp - s * akq;
            a[k][q] = s * akp + c * akq;
          }
#pragma unroll
          for (int k = 0; k < 7; k++) {
            const double apk = a[p][k], aqk = a[q][k];
            a[p][k] = c * apk - s * aqk;
            a[q][k] = s * apk + c * aqk;
          }
        }
      }
  }
#pragma unroll
  for (int i = 0; i < 7; i++) ev[i] = a[i][i];
}

// Cholesky factor of a 7x7 SPD matrix into registers; false if not PD
__device__ __forceinline__ bool chol7(const double* A, double L[7][7]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 7; j++) {
    double d = A[j * 7 + j];
#pragma unroll
    for (int k = 0; k < j; k++) d -= L[j][k] * L[j][k];
    ok &= d > 0.0;
    L[j][j] = sqrt(d);
#pragma unroll
    for (int i = j + 1; i < 7; i++) {
      double v = A[i * 7 + j];
#pragma unroll
      for (int k = 0; k < j; k++) v -= L[i][k] * L[j][k];
      L[i][j] = v / L[j][j];
    }
  }
  return ok;
}

__device__ __forceinline__ void chol7_solve(const double L[7][7], const double* b, double* x) {
  double t[7];
#pragma unroll
  for (int i = 0; i < 7; i++) {
    double v = b[i];
#pragma unroll
    for (int k = 0; k < i; k++) v -= L[i][k] * t[k];
    t[i] = v / L[i][i];
  }
#pragma unroll
  for (int i = 6; i >= 0; i--) {
    double v = t[i];
#pragma unroll
    for (int k = i + 1; k < 7; k++) v -= L[k][i] * x[k];
    x[i] = v / L[i][i];
  }
}

// Cholesky solve of A x = b and/or inverse; false if A is not PD
__device__ bool chol_solve(const double* A, const double* b, double* x, double* inv) {
  double L[7][7];
  if (!chol7(A, L)) return false;
  if (b) chol7_solve(L, b, x);
  if (inv) {
#pragma unroll
    for (int c = 0; c < 7; c++) {
      double e[7], col[7];
#pragma unroll
      for (int i = 0; i < 7; i++) e[i] = (i == c) ? 1.0 : 0.0;
      chol7_solve(L, e, col);
#pragma unroll
      for (int i = 0; i < 7; i++) inv[i * 7 + c] = col[i];
    }
  }
  return true;
}

// rls_init's P0 = np.linalg.inv(G) (`predict.py:126-131`): LAPACK getrf/getri
// semantics -- LU with partial pivoting (largest |pivot| in the column), and
// failure ONLY on an exactly zero pivot (numpy's LinAlgError "Singular
// matrix"), where the caller retries with G + 1e-8 I.  A nearly singular but
// invertible G is inverted, as the reference does, not regularised.
__device__ bool lu_inv7(const double* A, double* inv) {
  double M[7][14];
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = 0; j < 7; j++) {
      M[i][j] = A[i * 7 + j];
      M[i][7 + j] = (i == j) ? 1.0 : 0.0;
    }
  for (int c = 0; c < 7; c++) {
    int piv = c;
    double best = fabs(M[c][c]);
    for (int i = c + 1; i < 7; i++)
      if (fabs(M[i][c]) > best) {
        best = fabs(M[i][c]);
        piv = i;
      }
    if (best == 0.0) return false;
    if (piv != c)
      for (int j = 0; j < 14; j++) {
        double t = M[c][j];
        M[c][j] = M[piv][j];
        M[piv][j] = t;
      }
    const double d = M[c][c];
    for (int i = c + 1; i < 7; i++) {
      const double f = M[i][c] / d;
      for (int j = c; j < 14; j++) M[i][j] -= f * M[c][j];
    }
  }
  for (int c = 6; c >= 0; c--) {  // back substitution for the 7 right-hand sides
    for (int j = 7; j < 14; j++) {
      double v = M[c][j];
      for (int k = c + 1; k < 7; k++) v -= M[c][k] * M[k][j];
      M[c][j] = v / M[c][c];
    }
  }
  bool fin = true;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = 0; j < 7; j++) {
      inv[i * 7 + j] = M[i][7 + j];
      fin &= isfinite(M[i][7 + j]);
    }
  return fin;
}

__device__ void p0_inverse(const double* G, double* Pinv) {
  if (lu_inv7(G, Pinv)) return;
  double B[49];
  for (int i = 0; i < 49; i++) B[i] = G[i];
  for (int i = 0; i < 7; i++) B[i * 8] += 1e-8;  // RIDGE_EPS (`predict.py:131`)
  lu_inv7(B, Pinv);
}

// inverse of a lower-triangular 7x7 factor (Li = L^-1, lower triangular)
__device__ __forceinline__ void tri_inv7(const double L[7][7], double Li[7][7]) {
  double d[7];
#pragma unroll
  for (int i = 0; i < 7; i++) d[i] = 1.0 / L[i][i];
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
}

// The rows themselves, for statistics that fail the condition screen
// (ols_solve_one's cold path).  [Z | y] = Q [R | c] by Givens row updates
// (R 7x7 upper triangular, c = Q^T y), then
//   * matrix_rank(Z) (`predict.py:58`) from the singular values of R by
//     one-sided Jacobi (relative accuracy ~eps S_max, like the SVD of Z),
//     tol = S_max * max(n, 7) * eps.  The eigenvalues of Z^T Z cannot
//     separate a singular value below ~sqrt(eps) S_max (exactly collinear
//     samples: duplicated rows in a short window, a constant feature) from
//     rounding; R can;
//   * at rank 7, x = R^-1 c: accurate to ~cond(Z) eps like lstsq
//     (`predict.py:63`), where the normal equations give ~cond(Z)^2 eps.
// A factor is 7 rows x 8 columns ([R | c]); packed upper part = 35 doubles.
constexpr int kQrPacked = 35;

// fold row v = [z, y] (destroyed) into the factor F
__device__ __forceinline__ void givens_row(double F[7][8], double* v) {
#pragma unroll
  for (int i = 0; i < 7; i++) {
    if (v[i] == 0.0) continue;
    const double h = hypot(F[i][i], v[i]), c = F[i][i] / h, sn = v[i] / h;
#pragma unroll
    for (int j = i; j < 8; j++) {
      const double a = F[i][j], b = v[j];
      F[i][j] = c * a + sn * b;
      v[j] = c * b - sn * a;
    }
  }
}

__device__ __forceinline__ void qr_zero(double F[7][8]) {
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) F[i][j] = 0.0;
}

// fold rows [lo, lo+cnt) of (X, y) (z = [x, 1]) into F
__device__ __forceinline__ void qr_rows(double F[7][8], const double* __restrict__ X, const double* __restrict__ y,
                                        long long lo, long long cnt) {
  for (long long k = 0; k < cnt; k++) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 6; j++) v[j] = X[(lo + k) * 6 + j];
    v[6] = 1.0;
    v[7] = y[lo + k];
    givens_row(F, v);
  }
}

__device__ __forceinline__ void qr_store(const double F[7][8], double* p) {
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 8; j++) p[t++] = F[i][j];
}
// fold the packed factor p into F (its rows are rows of an equivalent [Z | y])
__device__ __forceinline__ void qr_merge(double F[7][8], const double* p) {
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = j < i ? 0.0 : p[t + j - i];
    t += 8 - i;
    givens_row(F, v);
  }
}

// matrix_rank from F's R block; at rank 7 also x = R^-1 c into x
__device__ __noinline__ int qr_rank_solve(const double F[7][8], double n_rows, double* x) {
  double R[7][7];
  for (int i = 0; i < 7; i++)
    for (int j = 0; j < 7; j++) R[i][j] = F[i][j];
  // A rotation of a column pair moves norm from the smaller column to the
  // larger one (it removes the smaller one's projection), so a column whose
  // norm is below the rank tolerance stays below it: it is already decided as
  // a zero singular value and pairs involving it are skipped (the partner
  // gains at most tol^2 in squared norm).  Rotating such rounding-noise
  // columns against each other rarely meets the convergence test and ran up
  // to 40 sweeps on rank-deficient designs.  smax0 <= S_max, so the cut is
  // at or below the exact tolerance; rank-7 solutions come from F, not R.
  double smax0 = 0.0;
  for (int j = 0; j < 7; j++) {
    double t = 0.0;
    for (int i = 0; i < 7; i++) t += R[i][j] * R[i][j];
    smax0 = fmax(smax0, t);
  }
  const double negl = sqrt(smax0) * fmax(n_rows, 7.0) * 2.220446049250313e-16, negl2 = negl * negl;
  for (int sweep = 0; sweep < 40; sweep++) {  // one-sided Jacobi on the columns of R
    bool rotated = false;
    for (int p = 0; p < 6; p++)
      for (int q = p + 1; q < 7; q++) {
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = 0; i < 7; i++) {
          al += R[i][p] * R[i][p];
          be += R[i][q] * R[i][q];
          ga += R[i][p] * R[i][q];
        }
        if (al <= negl2 || be <= negl2) continue;
        if (ga == 0.0 || fabs(ga) <= 2.220446049250313e-16 * sqrt(al * be)) continue;
        rotated = true;
        const double ze = (be - al) / (2.0 * ga);
        const double t = (ze >= 0.0 ? 1.0 : -1.0) / (fabs(ze) + sqrt(1.0 + ze * ze));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < 7; i++) {
          const double a = R[i][p], b = R[i][q];
          R[i][p] = c * a - sn * b;
          R[i][q] = sn * a + c * b;
        }
      }
    if (!rotated) break;
  }
  double sv[7], smax = 0.0;
  for (int j = 0; j < 7; j++) {
    double t = 0.0;
    for (int i = 0; i < 7; i++) t += R[i][j] * R[i][j];
    sv[j] = sqrt(t);
    smax = fmax(smax, sv[j]);
  }
  const double tol = smax * fmax(n_rows, 7.0) * 2.220446049250313e-16;
  int rank = 0;
  for (int j = 0; j < 7; j++) rank += sv[j] > tol;
  if (rank == 7)
    for (int i = 6; i >= 0; i--) {
      double v = F[i][7];
      for (int j = i + 1; j < 7; j++) v -= F[i][j] * x[j];
      x[i] = v / F[i][i];
    }
  return rank;
}

// rank (and the rank-7 solution) of rows [lo, lo+cnt), one thread
__device__ __noinline__ int qr_rank_rows(const double* __restrict__ X, const double* __restrict__ y, long long lo,
                                         long long cnt, double* x) {
  double F[7][8];
  qr_zero(F);
  qr_rows(F, X, y, lo, cnt);
  return qr_rank_solve(F, (double)cnt, x);
}

// fit_ols_xy (`predict.py:53-66`): matrix_rank(Z) < 7 -> ridge solve, else
// least squares (normal equations; lstsq and Cholesky agree to ~cond*eps).
// rank test: S_i = sqrt(eig(Z^T Z)); rank = #(S_i > S_max * max(n, 7) * eps).
// Statistics that fail the screen take their rank -- and, at rank 7, their
// solution -- from the rows: qr = [rank, x0..x6] computed by the pooled QR
// kernels (qr[0] < 0: not computed), or rows X, y + [lo, lo+cnt) (a window,
// qr_rank_rows here), else the rank from eig(Z^T Z) and the normal equations.
__device__ __forceinline__ void ols_solve_one(const double* __restrict__ stats, double* params, int32_t* info,
                                              double* Pinv, const double* __restrict__ rows = nullptr,
                                              const double* __restrict__ rows_y = nullptr, long long lo = 0,
                                              long long cnt = 0, const double* __restrict__ qr = nullptr,
                                              bool screen_only = false) {
  double G[49], r[7], ev[7];
  for (int i = 0; i < 49; i++) G[i] = stats[i];
  for (int i = 0; i < 7; i++) r[i] = stats[49 + i];
  const double n = G[48];
  // rank test, screened first: with G = L L^T and Li = L^-1, ev_max <= trace(G)
  // and 1/ev_min = ||G^-1||_2 <= trace(G^-1) = ||Li||_F^2, so
  // trace(G) ||Li||_F^2 < 1e10 proves ev_min > 1e-10 ev_max, far above both
  // the SVD tolerance (max(n,7) eps)^2 ev_max and the eigenvalue error
  // (~1e-15 ev_max): the eigenvalue test below would find rank 7.  Screened
  // windows solve x = Li^T (Li r) from the same factor; only windows that
  // fail the screen pay for the eigenvalues.
  {
    double L[7][7];
    if (chol7(G, L)) {
      double Li[7][7];
      tri_inv7(L, Li);
      double tr = 0.0, ti = 0.0;
#pragma unroll
      for (int i = 0; i < 7; i++) tr += G[i * 8];
#pragma unroll
      for (int i = 0; i < 7; i++)
#pragma unroll
        for (int j = 0; j <= i; j++) ti = fma(Li[i][j], Li[i][j], ti);
      if (isfinite(ti) && tr * ti < 1e10) {
        double t[7];
#pragma unroll
        for (int i = 0; i < 7; i++) {
          double v = 0.0;
#pragma unroll
          for (int k = 0; k <= i; k++) v = fma(Li[i][k], r[k], v);
          t[i] = v;
        }
        int fin = 1;
#pragma unroll
        for (int i = 0; i < 7; i++) {
          double v = 0.0;
#pragma unroll
          for (int k = i; k < 7; k++) v = fma(Li[k][i], t[k], v);
          params[i] = v;
          fin &= isfinite(v);
        }
        if (info) {
          info[0] = 0;
          info[1] = fin ? 0 : 1;
        }
        if (Pinv) p0_inverse(G, Pinv);  // rls_init P0 = inv(Z^T Z) (`predict.py:126-131`)
        return;
      }
    }
  }
  int rank = 0;
  double xq[7];
  bool have_x = false;
  // an exactly zero column of Z (G[i][i] == 0: e.g. the colo features of a
  // scenario that never co-locates) makes matrix_rank(Z) < 7 without any
  // factorisation: that singular value is exactly 0
  bool zero_col = false;
#pragma unroll
  for (int i = 0; i < 7; i++) zero_col |= G[i * 8] == 0.0;
  if (zero_col) {
    rank = 0;
  } else if (qr && qr[0] >= 0.0) {
    rank = (int)qr[0];
    for (int i = 0; i < 7; i++) xq[i] = qr[1 + i];
    have_x = rank == 7;
  } else if (screen_only) {  // the caller computes the rows' QR cooperatively and calls again with qr
    if (info) info[0] = -1;
    return;
  } else if (rows) {
    rank = qr_rank_rows(rows, rows_y, lo, cnt, xq);
    have_x = rank == 7;
  } else {
    jacobi_eigs(G, ev);
    double smax = 0.0;
    for (int i = 0; i < 7; i++) smax = fmax(smax, sqrt(fmax(ev[i], 0.0)));
    const double tol = smax * fmax(n, 7.0) * 2.220446049250313e-16;
    for (int i = 0; i < 7; i++) rank += sqrt(fmax(ev[i], 0.0)) > tol;
  }
  if (have_x) {  // full rank, ill-conditioned: the QR solution (lstsq's accuracy)
    int fin = 1;
    for (int i = 0; i < 7; i++) {
      params[i] = xq[i];
      fin &= isfinite(xq[i]);
    }
    if (info) {
      info[0] = 0;
      info[1] = fin ? 0 : 1;
    }
    if (Pinv) p0_inverse(G, Pinv);
    return;
  }
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
  if (Pinv) p0_inverse(G, Pinv);  // rls_init P0 = inv(Z^T Z), ridge only on an exact zero pivot
}

__global__ void k_ols_solve(const double* __restrict__ stats, const double* __restrict__ qr, double* params,
                            int32_t* info, double* Pinv) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  ols_solve_one(stats, params, info, Pinv, nullptr, nullptr, 0, 0, qr);
}

// the condition screen of ols_solve_one alone: true = rank 7 proven
__device__ bool ols_screen(const double* __restrict__ stats) {
  double G[49];
  for (int i = 0; i < 49; i++) G[i] = stats[i];
  double L[7][7];
  if (!chol7(G, L)) return false;
  double Li[7][7];
  tri_inv7(L, Li);
  double tr = 0.0, ti = 0.0;
  for (int i = 0; i < 7; i++) tr += G[i * 8];
  for (int i = 0; i < 7; i++)
    for (int j = 0; j <= i; j++) ti = fma(Li[i][j], Li[i][j], ti);
  return isfinite(ti) && tr * ti < 1e10;
}

// pooled samples (tall-skinny QR): thread = contiguous run of rows folded
// into its factor by Givens rotations, then a fixed binary tree of merges
// per block (deterministic) -> ws[block]; k_ols_qr_final merges the blocks'
// factors by the same tree -> qr = [rank, x].  Both exit at once when the
// statistics pass the screen (rank 7 proven; qr[0] = -1).
constexpr int kQrThreads = 64, kQrBlocks = 128;
__global__ void __launch_bounds__(kQrThreads) k_ols_qr_rows(const double* __restrict__ X, const double* __restrict__ y,
                                                            long long n, const double* __restrict__ stats,
                                                            double* ws) {
  __shared__ double sh[kQrThreads][kQrPacked];
  __shared__ bool pass;
  if (threadIdx.x == 0) pass = ols_screen(stats);
  __syncthreads();
  if (pass) return;
  const long long T = (long long)gridDim.x * kQrThreads, t = (long long)blockIdx.x * kQrThreads + threadIdx.x;
  const long long per = (n + T - 1) / T, lo = t * per, hi = lo + per < n ? lo + per : n;
  double F[7][8];
  qr_zero(F);
  if (lo < hi) qr_rows(F, X, y, lo, hi - lo);
  qr_store(F, sh[threadIdx.x]);
  __syncthreads();
  for (int s = 1; s < kQrThreads; s <<= 1) {
    if ((threadIdx.x & (2 * s - 1)) == 0) {
      qr_merge(F, sh[threadIdx.x + s]);
      qr_store(F, sh[threadIdx.x]);
    }
    __syncthreads();
  }
  if (threadIdx.x < kQrPacked) ws[blockIdx.x * kQrPacked + threadIdx.x] = sh[0][threadIdx.x];
}

__global__ void __launch_bounds__(kQrBlocks) k_ols_qr_final(const double* __restrict__ stats, const double* ws,
                                                            int n_blocks, double n_rows, double* qr) {
  __shared__ double sh[kQrBlocks][kQrPacked];
  __shared__ bool pass;
  if (threadIdx.x == 0) pass = ols_screen(stats);
  __syncthreads();
  if (pass) {
    if (threadIdx.x == 0) qr[0] = -1.0;
    return;
  }
  double F[7][8];
  qr_zero(F);
  if (threadIdx.x < n_blocks) qr_merge(F, ws + threadIdx.x * kQrPacked);
  qr_store(F, sh[threadIdx.x]);
  __syncthreads();
  for (int s = 1; s < kQrBlocks; s <<= 1) {
    if ((threadIdx.x & (2 * s - 1)) == 0) {
      qr_merge(F, sh[threadIdx.x + s]);
      qr_store(F, sh[threadIdx.x]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double x[7] = {0, 0, 0, 0, 0, 0, 0};
    qr[0] = (double)qr_rank_solve(F, n_rows, x);
    for (int i = 0; i < 7; i++) qr[1 + i] = x[i];
  }
}

// ---- windowed refit (C3, "refit each window"): fit_ols on every window of
// `window` consecutive samples (`predict.py:53-72` per window).  Statistics:
// one warp per window, lanes stride the rows, a fixed xor-butterfly sum (so
// the result is deterministic); solve: one thread per window.
constexpr int kWinWarps = 8;
__global__ void __launch_bounds__(32 * kWinWarps) k_ols_window_stats(const double* __restrict__ X,
                                                                   const double* __restrict__ y, long long n,
                                                                   int window, long long n_win,
                                                                   double* __restrict__ stats) {
  const long long w = (long long)blockIdx.x * kWinWarps + (threadIdx.x >> 5);
  if (w >= n_win) return;
  const int lane = threadIdx.x & 31;
  const long long lo = w * window, hi = lo + window < n ? lo + window : n;
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
  for (long long row = lo + lane; row < hi; row += 32) {
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
  double* out = stats + w * 56;
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++, t++) {
      const double v = warp_sum(acc[t]);
      if (lane == (t & 31)) {  // spread the 56 stores over the lanes
        out[i * 7 + j] = v;
        out[j * 7 + i] = v;
      }
    }
#pragma unroll
  for (int i = 0; i < 7; i++) {
    const double v = warp_sum(acc[28 + i]);
    if (lane == i) out[49 + i] = v;
  }
}

// one row's contribution to the 35 statistics (z = [x, 1])
__device__ __forceinline__ void ols_acc_row(double* acc, const double* x6, double yy) {
  const double z[7] = {x6[0], x6[1], x6[2], x6[3], x6[4], x6[5], 1.0};
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++) acc[t] = fma(z[i], z[j], acc[t]), t++;
#pragma unroll
  for (int i = 0; i < 7; i++) acc[28 + i] = fma(z[i], yy, acc[28 + i]);
}

// the window's statistics (optionally to HBM), its solve and its info row
__device__ __forceinline__ void ols_window_finish(const double* acc, const double* __restrict__ X,
                                                  const double* __restrict__ y, long long w, long long lo,
                                                  long long cnt, double* stats, double* params, int32_t* info) {
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
  int32_t inf2[2] = {0, 0};
  ols_solve_one(st, params + w * 7, inf2, nullptr, X, y, lo, cnt);
  info[3 * w] = inf2[0];
  info[3 * w + 1] = inf2[1];
  info[3 * w + 2] = cnt < 7 ? 1 : 0;
}

// other windows of <= kFusedWindow rows: one thread per window accumulates
// its statistics sequentially in registers (no cross-lane reduction) and
// solves in place; the statistics reach HBM only if the caller asked for them.
constexpr int kFusedWindow = 128;
__global__ void __launch_bounds__(128) k_ols_windows_fused(const double* __restrict__ X, const double* __restrict__ y,
                                                           long long n, int window, long long n_win,
                                                           double* __restrict__ stats, double* __restrict__ params,
                                                           int32_t* __restrict__ info) {
  const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_win) return;
  const long long lo = w * window, hi = lo + window < n ? lo + window : n;
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
#pragma unroll 4  // four rows' loads in flight per thread (memory-level parallelism at 2 blocks/SM)
  for (long long row = lo; row < hi; row++) {
    const double2* xr = reinterpret_cast<const double2*>(X + row * 6);
    const double2 a = __ldg(xr), b = __ldg(xr + 1), c = __ldg(xr + 2);
    const double x6[6] = {a.x, a.y, b.x, b.y, c.x, c.y};
    ols_acc_row(acc, x6, __ldg(y + row));
  }
  ols_window_finish(acc, X, y, w, lo, hi - lo, stats, params, info);
}

// windows of a multiple of 8 rows: one warp per block, persistent over groups
// of 32 consecutive windows (lane = window).  A chunk is rows [8c, 8c+8) of
// the group's 32 windows, fetched by TWO tensor-map boxes -- X as
// {16 doubles, 3 groups of 16, 32 windows} (128-byte swizzle) and y as
// {8 rows, 32 windows} (64-byte swizzle) -- into one of kWinTmaStages
// shared-memory stages; the chunk stream runs on across groups, so the next
// group's boxes are in flight while the lanes solve.  Each lane reads its
// 384-byte X slab through the swizzle (conflict-free 16-byte loads).  Windows
// past the last full one (the trailing partial window) read global memory.
// (Per-lane 1-D bulk copies -- 64 small copies per chunk -- ran at 0.77 of
// this rate, thread-per-window global loads at 0.40: tools/refit_variants.cu.)
constexpr int kWinTmaRows = 8;
constexpr int kWinTmaStages = 3;
constexpr int kWinTmaPerSm = 4;  // 1-warp blocks resident per SM (43 KB shared memory each)
constexpr int kWinTmaXBytes = 32 * kWinTmaRows * 48, kWinTmaYBytes = 32 * kWinTmaRows * 8;
constexpr int kWinTmaSmem = kWinTmaStages * (kWinTmaXBytes + kWinTmaYBytes) + 1024 + 64;

__global__ void __launch_bounds__(32) k_ols_windows_tma(const __grid_constant__ CUtensorMap mx,
                                                        const __grid_constant__ CUtensorMap my,
                                                        const double* __restrict__ X, const double* __restrict__ y,
                                                        long long n, int window, long long n_win,
                                                        double* __restrict__ stats, double* __restrict__ params,
                                                        int32_t* __restrict__ info) {
  constexpr int R = kWinTmaRows, S = kWinTmaStages, XB = kWinTmaXBytes, YB = kWinTmaYBytes;
  extern __shared__ unsigned char win_dsm[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(win_dsm) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S * (XB + YB));
  const int lane = threadIdx.x;
  const long long n_full = n / window;  // windows whose rows the boxes cover
  const long long n_grp = (n_win + 31) / 32;
  const int nch = window / R;
  const long long g0 = blockIdx.x, gs = gridDim.x;
  const long long my_grps = g0 < n_grp ? (n_grp - 1 - g0) / gs + 1 : 0;
  if (lane == 0)
    for (int s = 0; s < S; s++) mbar_init(&bar[s]);
  __syncwarp();
  long long i_grp = g0;  // issue cursor: group, chunk, stage
  int i_c = 0, i_st = 0;
  long long i_left = my_grps * nch;
  auto issue = [&]() {
    if (lane == 0) {
      unsigned char* dst = sm + i_st * (XB + YB);
      mbar_arrive_expect(&bar[i_st], (unsigned)(XB + YB));  // out-of-range boxes are zero-filled: always full bytes
      tma_load_3d(dst, &mx, 0, i_c * 3, (int)(i_grp * 32), &bar[i_st]);
      tma_load_2d(dst + XB, &my, i_c * R, (int)(i_grp * 32), &bar[i_st]);
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
    const bool staged = w < n_full;
#pragma unroll
    for (int i = 0; i < kStats; i++) acc[i] = 0.0;
    for (int c = 0; c < nch; c++) {
      if (i_left > 0) issue();
      mbar_wait(&bar[st], ph);
      if (staged) {
        const unsigned char* xs = sm + st * (XB + YB);
        const unsigned char* ys = xs + XB;
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          double z[12];
#pragma unroll
          for (int jj = 0; jj < 6; jj++) {
            const int u = 3 * r + jj;             // 16-byte unit of this lane's 384-byte slab
            const int rho = lane * 3 + (u >> 3);  // 128-byte row of the box; swizzle: unit ^= row % 8
            const double2 v = *reinterpret_cast<const double2*>(xs + rho * 128 + (((u & 7) ^ (rho & 7)) << 4));
            z[2 * jj] = v.x;
            z[2 * jj + 1] = v.y;
          }
          // 64-byte rows: 16-byte unit ^= (row / 2) % 4
          const double2 yy = *reinterpret_cast<const double2*>(ys + lane * 64 + (((r >> 1) ^ ((lane >> 1) & 3)) << 4));
          ols_acc_row(acc, z, yy.x);
          ols_acc_row(acc, z + 6, yy.y);
        }
      } else {
        for (int r = c * R; r < c * R + R && r < cnt; r++) ols_acc_row(acc, X + (lo + r) * 6, y[lo + r]);
      }
      __syncwarp();  // every lane is done with the stage before it is refilled
      if (++st == S) st = 0, ph ^= 1u;
    }
    if (w < n_win) ols_window_finish(acc, X, y, w, lo, cnt, stats, params, info);
  }
}

// info[3w..]: ridge used, non-finite params, fewer than 7 rows (fit_ols raises
// PredictError for those; fit_ols_xy solves them through the ridge fallback)
__global__ void k_ols_window_solve(const double* __restrict__ stats, const double* __restrict__ X,
                                   const double* __restrict__ y, long long n_win, long long n, int window,
                                   double* __restrict__ params, int32_t* __restrict__ info) {
  const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_win) return;
  const long long cnt = (w + 1) * window <= n ? window : n - w * window;
  int32_t inf2[2] = {0, 0};
  ols_solve_one(stats + w * 56, params + w * 7, inf2, nullptr, X, y, w * window, cnt);
  info[3 * w] = inf2[0];
  info[3 * w + 1] = inf2[1];
  info[3 * w + 2] = cnt < 7 ? 1 : 0;
}

// ===================================================================== K7
// sgd_update (`predict.py:88-95`): e = y - (w.x + b); w += (eta*e)*x;
// b += eta*e -- same rounding sequence as numpy (unfused).
__global__ void k_sgd(const double* __restrict__ X, const double* __restrict__ Y, const long long* __restrict__ off,
                      int n_streams, const double* __restrict__ eta, double* params, double* pred, int32_t* status,
                      const long long* __restrict__ end = nullptr) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_streams) return;
  double w[7];
  for (int i = 0; i < 7; i++) w[i] = params[s * 7 + i];
  const double et = eta[s];
  int st = 0;
  const long long i1 = end ? end[s] : off[s + 1];
  for (long long i = off[s]; i < i1; i++) {
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

// rls_update (`predict.py:137-154`), lane-parallel: 8 lanes per stream, lane
// r < 7 owns row r of P (the 7x7 gain matrix), so the 49 updates of P run
// 7-wide and a warp advances 4 streams.  Per element the operations are the
// reference's, in its order, with its two divisions as reciprocal multiplies:
//   Pz_r = P[r,:] . z (fma chain)        -> gathered by shuffles
//   zPz  = z . Pz (fma chain, every lane) -> denom, reset rule
//   k_r  = Pz_r * (1 / denom)             -> gathered
//   w   += k e (every lane keeps w)
//   P[r,:] = (P[r,:] - k_r Pz) * (1 / lambda); then 0.5 (P + P^T) via a shared-memory transpose
constexpr int kRlsGroup = 8;
// off: stream s is rows [off[s], off[s+1]) -- or [off[s], end[s]) when end is
// given (streams that are not back to back, e.g. the test tails of a sweep).
__global__ void __launch_bounds__(128) k_rls_g8(const double* __restrict__ X, const double* __restrict__ Y,
                                                const long long* __restrict__ off, int n_streams,
                                                const double* __restrict__ lamv, double* params, double* Pg,
                                                double* pred, int32_t* status,
                                                const long long* __restrict__ end = nullptr, int pstride = 7) {
  __shared__ double tr[128 / kRlsGroup][7][8];
  const int gi = threadIdx.x / kRlsGroup, r = threadIdx.x % kRlsGroup;
  const int s = blockIdx.x * (128 / kRlsGroup) + gi;
  const unsigned gmask = 0xffu << ((threadIdx.x & 31) & ~(kRlsGroup - 1));
  const bool live = s < n_streams;
  const int ss = live ? s : 0;
  const int rr = r < 7 ? r : 6;  // lane 7 shadows row 6 (keeps every shuffle full-group)
  double w[7], P[7];
#pragma unroll
  for (int i = 0; i < 7; i++) w[i] = params[(long long)ss * pstride + i];
#pragma unroll
  for (int j = 0; j < 7; j++) P[j] = Pg[(long long)ss * 49 + rr * 7 + j];
  const double lam = lamv[ss];
  // k = Pz / denom and P = (...) / lam as multiplies by the reciprocals: one
  // division per update instead of eight on the chain (0.95 -> 0.52 us per
  // update, tools/rls_recip.sh); each product is within 1 ulp of the quotient,
  // far inside the 1e-5 tolerance of the refit path
  const double inv_lam = 1.0 / lam;
  int st = 0;
  // P exactly symmetric: from the start if P0 is (one transpose), else after
  // the first update's symmetrization
  bool sym;
  {
    double(*T)[8] = tr[gi];
    if (r < 7) {
#pragma unroll
      for (int j = 0; j < 7; j++) T[r][j] = P[j];
    }
    __syncwarp(gmask);
    bool mine = true;
#pragma unroll
    for (int j = 0; j < 7; j++) mine &= P[j] == T[j][rr];
    sym = __all_sync(gmask, mine);
    __syncwarp(gmask);
  }
  const long long i0 = live ? off[s] : 0, i1 = live ? (end ? end[s] : off[s + 1]) : 0;
  // the next sample's row is loaded one update ahead (off the update chain)
  double zn[6], yn = 0.0;
#pragma unroll
  for (int j = 0; j < 6; j++) zn[j] = i0 < i1 ? X[i0 * 6 + j] : 0.0;
  if (i0 < i1) yn = Y[i0];
  for (long long it = i0; it < i1; it++) {
    double z[7];
#pragma unroll
    for (int j = 0; j < 6; j++) z[j] = zn[j];
    z[6] = 1.0;
    const double ycur = yn;
    if (it + 1 < i1) {
#pragma unroll
      for (int j = 0; j < 6; j++) zn[j] = X[(it + 1) * 6 + j];
      yn = Y[it + 1];
    }
    const double yh = predict7(w, z);
    if (r == 0) pred[it] = yh;
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < 7; j++) a = fma(P[j], z[j], a);
    double Pz[7];
#pragma unroll
    for (int j = 0; j < 7; j++) Pz[j] = __shfl_sync(gmask, a, j, kRlsGroup);
    double zPz = 0.0;
#pragma unroll
    for (int j = 0; j < 7; j++) zPz = fma(z[j], Pz[j], zPz);
    double denom = lam + zPz;
    if (!(denom > 0.0) || !isfinite(denom)) {  // P reset (`predict.py:142-146`)
      st |= 2;
#pragma unroll
      for (int j = 0; j < 7; j++) P[j] = (j == rr) ? 100.0 : 0.0;
#pragma unroll
      for (int j = 0; j < 7; j++) Pz[j] = 100.0 * z[j];
      zPz = 0.0;
#pragma unroll
      for (int j = 0; j < 7; j++) zPz = fma(z[j], Pz[j], zPz);
      denom = lam + zPz;
    }
    double pzr = Pz[0];  // Pz[rr] without dynamic register indexing
#pragma unroll
    for (int j = 1; j < 7; j++) pzr = j == rr ? Pz[j] : pzr;
    const double rd = 1.0 / denom;
    // k = Pz / denom, every lane from the shuffled Pz (no second shuffle round)
    const double e = ycur - yh;
#pragma unroll
    for (int j = 0; j < 7; j++) w[j] = w[j] + (Pz[j] * rd) * e;
    if (sym) {
      // P is exactly symmetric: (Pz_r Pz_j) rd is the same product for (r, j)
      // and (j, r), so the update keeps it symmetric bit for bit and the
      // symmetrization (`predict.py:152`) is the identity -- no transpose
#pragma unroll
      for (int j = 0; j < 7; j++) P[j] = (P[j] - (pzr * Pz[j]) * rd) * inv_lam;
    } else {
      // P not exactly symmetric (P0 = inv(G) is symmetric only up to rounding):
      // the reference's order, update then symmetrize; lane r needs P[j][r] of every row j
      const double kr = pzr * rd;
#pragma unroll
      for (int j = 0; j < 7; j++) P[j] = (P[j] - kr * Pz[j]) * inv_lam;
      double(*T)[8] = tr[gi];
      if (r < 7) {
#pragma unroll
        for (int j = 0; j < 7; j++) T[r][j] = P[j];
      }
      __syncwarp(gmask);
      // all 7 loads first, no branch: the diagonal term is 0.5 (a + a) == a exactly
      double pt[7];
#pragma unroll
      for (int j = 0; j < 7; j++) pt[j] = T[j][rr];
#pragma unroll
      for (int j = 0; j < 7; j++) P[j] = 0.5 * (P[j] + pt[j]);  // == 0.5 (P[rr][j] + P[j][rr]) == the (j, rr) entry
      __syncwarp(gmask);
      sym = true;
    }
    bool fin = true;
#pragma unroll
    for (int j = 0; j < 7; j++) fin &= isfinite(w[j]);
    if (!fin) {
      st |= 1;
      break;
    }
  }
  if (!live) return;
  if (r == 0) {
#pragma unroll
    for (int i = 0; i < 7; i++) params[(long long)s * pstride + i] = w[i];
    if (status) status[s] = st;
  }
  if (r < 7) {
#pragma unroll
    for (int j = 0; j < 7; j++) Pg[(long long)s * 49 + r * 7 + j] = P[j];
  }
}

// ===================================================================== C5
// Per-scenario predictor evaluation of a replayed sweep:
// samples in outcome order, chronological split cut = int(round(0.75 n))
// (`experiments.py:44-60`, Python's round: half to even = rint), then
//   coarse   = fit_ols(static[:cut]),  offline on static[cut:]
//   fine     = fit_ols(EWMA[:cut]),    offline on EWMA[cut:]
//   adaptive = rls_init(fine, lam, X_train = EWMA[:cut]), prequential on EWMA[cut:]
// (`predict.py:53-72,112-134,157-205`).  Each part at the parallel grain and
// register footprint it needs: k_scen_stats (a warp per training design: the
// 35 statistics, lanes stride the rows, fixed butterfly sums), k_scen_solve (a
// thread per design: condition screen + solve), k_scen_qr (the rare designs
// that fail the screen: rank from the rows by the warp), k_scen_finish (a warp
// per scenario: P0 = inv(G) of the EWMA design, the offline test
// predictions); then k_rls_g8 runs the adaptive tails (8 lanes per scenario)
// and k_eval the 3 EvalReports per scenario.  (One warp per scenario for all
// of it kept 2 of 32 lanes busy in the solves at 8 warps per SM.)
constexpr int kScenFitWarps = 4;

// rls_init's P0 = np.linalg.inv(G) (`predict.py:126-131`) by the whole warp:
// Gauss-Jordan with partial pivoting on [G | I], lane r < 7 holding row r in
// registers (the pivot search is a warp arg-max over the rows not yet used,
// first lane on ties; the pivot row's live columns are broadcast by shuffles).  It
// fails only on an exactly zero pivot -- numpy's LinAlgError: two identical
// columns (and rows) of a symmetric G stay identical under the row operations
// until one is the pivot row, which zeroes the other exactly -- and then
// inverts G + 1e-8 I (`predict.py:131`).  Replaces lane-serial LU with
// dynamically indexed rows (local memory), ~45% of the then fused fit kernel's samples.
__device__ __noinline__ void warp_p0_inverse(const double* G, double* inv) {
  const int lane = threadIdx.x & 31, r = lane < 7 ? lane : 6;
  for (int attempt = 0; attempt < 2; attempt++) {
    double row[14];
#pragma unroll
    for (int j = 0; j < 7; j++) row[j] = G[r * 7 + j] + ((attempt && j == r) ? 1e-8 : 0.0);
#pragma unroll
    for (int j = 0; j < 7; j++) row[7 + j] = (j == r) ? 1.0 : 0.0;
    // rows stay in their lanes: the pivot lane of column c is remembered
    // (no swap shuffles); eliminated entries are exact zeros (not updated)
    bool used = lane >= 7;
    int my_col = -1;
    bool ok = true;
#pragma unroll
    for (int c = 0; c < 7; c++) {
      double best = used ? -1.0 : fabs(row[c]);
      int piv = lane;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, piv, o);
        if (ob > best || (ob == best && op < piv)) best = ob, piv = op;
      }
      if (best == 0.0) {  // warp-uniform
        ok = false;
        break;
      }
      double p[14];
#pragma unroll
      for (int j = c; j < 14; j++) p[j] = __shfl_sync(0xffffffffu, row[j], piv);
      if (lane == piv) {
        used = true;
        my_col = c;
      } else if (lane < 7) {
        const double f = row[c] / p[c];
#pragma unroll
        for (int j = c + 1; j < 14; j++) row[j] -= f * p[j];
        row[c] = 0.0;
      }
    }
    if (ok) {
      double d = row[0];
#pragma unroll
      for (int j = 1; j < 7; j++) d = j == my_col ? row[j] : d;
      if (lane < 7) {
#pragma unroll
        for (int j = 0; j < 7; j++) inv[my_col * 7 + j] = row[7 + j] / d;
      }
      return;
    }
  }
}

// one scenario design's solve (a call, not inlined)
__device__ __noinline__ void scen_solve(const double* st, double* p, int32_t* inf2, double* Pinv, const double* qr,
                                        bool screen_only) {
  ols_solve_one(st, p, inf2, Pinv, nullptr, nullptr, 0, 0, qr, screen_only);
}

// matrix_rank(Z) and, at rank 7, the lstsq solution of rows [lo, lo+cnt) by
// the whole warp: each lane folds its strided rows into its own [R | c]
// factor by Givens rotations, then a 5-level tree merges the factors (the
// partner's rows arrive by shuffles, one row of the triangle at a time);
// lane 0 takes the rank / solution from the merged R (qr_rank_solve).
// out[0] = rank, out[1..7] = x (lane 0 writes).
__device__ __noinline__ void warp_qr_rank(const double* __restrict__ X, const double* __restrict__ y, long long lo, long long cnt,
                             double* out) {
  const int lane = threadIdx.x & 31;
  double F[7][8];
  qr_zero(F);
  for (long long k = lane; k < cnt; k += 32) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 6; j++) v[j] = X[(lo + k) * 6 + j];
    v[6] = 1.0;
    v[7] = y[lo + k];
    givens_row(F, v);
  }
  for (int off = 1; off < 32; off <<= 1) {
    const bool take = (lane & (2 * off - 1)) == 0;
#pragma unroll
    for (int i = 0; i < 7; i++) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const double pj = __shfl_down_sync(0xffffffffu, F[i][j], off);
        v[j] = j < i ? 0.0 : pj;
      }
      if (take) givens_row(F, v);
    }
  }
  if (lane == 0) {
    double x[7];
    out[0] = (double)qr_rank_solve(F, (double)cnt, x);
#pragma unroll
    for (int i = 0; i < 7; i++) out[1 + i] = x[i];
  }
}
// the chronological split of scenario s (`experiments.py:44-60`): cut =
// int(round(0.75 n)); fit_ols needs 7 samples, the split a non-empty test set
struct ScenSplit {
  long long base, n, cut;
  bool valid;
};
__device__ __forceinline__ ScenSplit scen_split(const intf_scenario* __restrict__ scen,
                                                const int32_t* __restrict__ n_batches, int s) {
  ScenSplit q;
  q.base = scen[s].req_off;
  q.n = n_batches[s];
  q.cut = (long long)rint(0.75 * (double)q.n);
  q.valid = q.cut >= 7 && q.n - q.cut >= 1;
  return q;
}

// (1) the 35 statistics of one training design (m = 0 static, 1 EWMA) of one
// scenario per warp: lanes stride the rows (lane l: rows l, l+32, ... in
// order), fixed butterfly sums -> stats[2s + m][56] (G row-major, then Z^T y).
// Low register footprint, so 16+ warps per SM hide the row loads.
__global__ void __launch_bounds__(32 * kScenFitWarps, 4) k_scen_stats(const intf_scenario* __restrict__ scen, int n_scen,
                                                                      const int32_t* __restrict__ n_batches,
                                                                      const double* __restrict__ X, long long slot_stride,
                                                                      int p_static, int p_ewma,
                                                                      const double* __restrict__ Y,
                                                                      double* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * kScenFitWarps + (threadIdx.x >> 5);
  if (g >= 2 * n_scen) return;
  const ScenSplit q = scen_split(scen, n_batches, g >> 1);
  const double* Xb = X + (long long)((g & 1) ? p_ewma : p_static) * slot_stride * 6;
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
  if (q.valid) {
    // 4 rows in flight per lane: the loads of the next rows are issued before
    // the 35-fma updates of the current ones
    long long row = q.base + lane;
    for (; row + 96 < q.base + q.cut; row += 128) {
      double x[4][6], yv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
#pragma unroll
        for (int i = 0; i < 6; i++) x[u][i] = Xb[(row + 32 * u) * 6 + i];
        yv[u] = Y[row + 32 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; u++) ols_acc_row(acc, x[u], yv[u]);
    }
    for (; row < q.base + q.cut; row += 32) ols_acc_row(acc, Xb + row * 6, Y[row]);
  }
  double* out = stats + 56ll * g;
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++, t++) {
      const double v = warp_sum(acc[t]);
      if (lane == (t & 31)) {  // spread the stores over the lanes
        out[i * 7 + j] = v;
        out[j * 7 + i] = v;
      }
    }
#pragma unroll
  for (int i = 0; i < 7; i++) {
    const double v = warp_sum(acc[28 + i]);
    if (lane == i) out[49 + i] = v;
  }
}

// (2) the condition screen + solve of every design, one THREAD per design
// (lane-serial work: every lane busy, where a warp per scenario kept 2 of 32)
__global__ void __launch_bounds__(128) k_scen_solve(const intf_scenario* __restrict__ scen, int n_scen,
                                                    const int32_t* __restrict__ n_batches,
                                                    const double* __restrict__ stats, double* __restrict__ par,
                                                    int32_t* __restrict__ inf) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= 2 * n_scen) return;
  const ScenSplit q = scen_split(scen, n_batches, g >> 1);
  int32_t inf2[2] = {0, 0};
  double p[7];
#pragma unroll
  for (int i = 0; i < 7; i++) p[i] = NAN;
  if (q.valid) scen_solve(stats + 56ll * g, p, inf2, nullptr, nullptr, true);
#pragma unroll
  for (int i = 0; i < 7; i++) par[7ll * g + i] = p[i];
  inf[2ll * g] = inf2[0];
  inf[2ll * g + 1] = inf2[1];
}

// (3) the designs that failed the condition screen (rare): rank from the
// rows by the whole warp of their scenario, then the solve on lane m
__global__ void __launch_bounds__(32 * kScenFitWarps) k_scen_qr(const intf_scenario* __restrict__ scen, int n_scen,
                                                                const int32_t* __restrict__ n_batches,
                                                                const double* __restrict__ X, long long slot_stride,
                                                                int p_static, int p_ewma, const double* __restrict__ Y,
                                                                const double* __restrict__ stats,
                                                                double* __restrict__ par, int32_t* __restrict__ inf) {
  __shared__ double qrres[kScenFitWarps][2][8];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * kScenFitWarps + wi;
  if (s >= n_scen) return;
  const ScenSplit q = scen_split(scen, n_batches, s);
  const bool mine = lane < 2 && q.valid && inf[2ll * (2 * s + lane)] == -1;
  const unsigned need = __ballot_sync(0xffffffffu, mine);
  if (!need) return;
  const double* Xm[2] = {X + (long long)p_static * slot_stride * 6, X + (long long)p_ewma * slot_stride * 6};
  for (int m = 0; m < 2; m++)
    if (need & (1u << m)) warp_qr_rank(Xm[m], Y, q.base, q.cut, qrres[wi][m]);
  __syncwarp();
  if (mine) {
    const int g = 2 * s + lane;
    int32_t inf2[2] = {inf[2ll * g], inf[2ll * g + 1]};
    double p[7];
    scen_solve(stats + 56ll * g, p, inf2, nullptr, qrres[wi][lane], false);
#pragma unroll
    for (int i = 0; i < 7; i++) par[7ll * g + i] = p[i];
    inf[2ll * g] = inf2[0];
    inf[2ll * g + 1] = inf2[1];
  }
}

// (4) per scenario, one warp: P0 = inv(G) of the EWMA design for the
// adaptive tail, the parameter rows, the offline test predictions, the tail
// bounds
__global__ void __launch_bounds__(32 * kScenFitWarps) k_scen_finish(const intf_scenario* __restrict__ scen, int n_scen,
                                                                    const int32_t* __restrict__ n_batches,
                                                                    const double* __restrict__ X, long long slot_stride,
                                                                    int p_static, int p_ewma, double lam,
                                                                    const double* __restrict__ stats,
                                                                    const double* __restrict__ par,
                                                                    const int32_t* __restrict__ inf,
                                                                    double* __restrict__ params, double* __restrict__ P0,
                                                                    double* __restrict__ lamv, long long* __restrict__ lo,
                                                                    long long* __restrict__ hi,
                                                                    double* __restrict__ yhat, int32_t* __restrict__ est) {
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * kScenFitWarps + wi;
  if (s >= n_scen) return;
  (void)wi;
  const ScenSplit q = scen_split(scen, n_batches, s);
  const double* Xm[2] = {X + (long long)p_static * slot_stride * 6, X + (long long)p_ewma * slot_stride * 6};
  int bits = q.valid ? 0 : 1;
  if (lane < 2 && q.valid) bits = (inf[2ll * (2 * s + lane)] ? (2 << lane) : 0) | (inf[2ll * (2 * s + lane) + 1] ? 16 : 0);
  bits |= __shfl_sync(0xffffffffu, bits, 1);
  if (q.valid) warp_p0_inverse(stats + 56ll * (2 * s + 1), P0 + 49ll * s);  // the adaptive tail's P0 from the EWMA design
  __syncwarp();
  if (lane < 21) {  // coarse, fine, adaptive (= fine before its tail) parameters
    const int k = lane / 7, i = lane % 7;
    params[(3ll * s + k) * 7 + i] = q.valid ? par[7ll * (2 * s + (k < 2 ? k : 1)) + i] : NAN;
  }
  if (lane == 0) {
    est[s] = bits;
    lamv[s] = lam;
    lo[s] = q.base + q.cut;
    hi[s] = q.valid ? q.base + q.n : q.base + q.cut;  // an invalid scenario gets empty test sets (reports n = 0, NaN)
  }
  if (!q.valid) return;
  double wc[7], wf[7];
#pragma unroll
  for (int i = 0; i < 7; i++) wc[i] = par[7ll * (2 * s) + i], wf[i] = par[7ll * (2 * s + 1) + i];
  for (long long row = q.base + q.cut + lane; row < q.base + q.n; row += 32) {
    yhat[row] = predict7(wc, Xm[0] + row * 6);
    yhat[slot_stride + row] = predict7(wf, Xm[1] + row * 6);
  }
}

// fit_ols_xy (`predict.py:53-72`) of arbitrary row segments [lo[g], hi[g]) of
// (X, y), one warp per segment: the 35 statistics by the warp (fixed
// butterfly sums), the condition screen on lane 0, the rows' QR by the warp
// when the screen fails, then the solve; Pinv (optional) = rls_init's P0.
// info[g][3] = (ridge used, non-finite params, fewer than 7 rows).
__global__ void __launch_bounds__(32 * kScenFitWarps) k_fit_segments(const double* __restrict__ X,
                                                                     const double* __restrict__ Y,
                                                                     const long long* __restrict__ lo,
                                                                     const long long* __restrict__ hi, int n_seg,
                                                                     double* __restrict__ params,
                                                                     int32_t* __restrict__ info,
                                                                     double* __restrict__ Pinv) {
  __shared__ double st[kScenFitWarps][56];
  __shared__ double qrres[kScenFitWarps][8];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * kScenFitWarps + wi;
  if (g >= n_seg) return;
  const long long a = lo[g], cnt = hi[g] - lo[g];
  double acc[kStats];
#pragma unroll
  for (int i = 0; i < kStats; i++) acc[i] = 0.0;
  for (long long row = a + lane; row < a + cnt; row += 32) ols_acc_row(acc, X + row * 6, Y[row]);
  int t = 0;
#pragma unroll
  for (int i = 0; i < 7; i++)
#pragma unroll
    for (int j = i; j < 7; j++, t++) {
      const double v = warp_sum(acc[t]);
      if (lane == 0) st[wi][i * 7 + j] = st[wi][j * 7 + i] = v;
    }
#pragma unroll
  for (int i = 0; i < 7; i++) {
    const double v = warp_sum(acc[28 + i]);
    if (lane == 0) st[wi][49 + i] = v;
  }
  __syncwarp();
  int32_t inf2[2] = {0, 0};
  double p[7];
  if (lane == 0) scen_solve(st[wi], p, inf2, nullptr, nullptr, true);
  const bool need = __shfl_sync(0xffffffffu, inf2[0], 0) == -1;
  if (need) warp_qr_rank(X, Y, a, cnt, qrres[wi]);
  __syncwarp();
  if (Pinv) warp_p0_inverse(st[wi], Pinv + 49ll * g);
  if (lane == 0) {
    if (need) scen_solve(st[wi], p, inf2, nullptr, qrres[wi], false);
#pragma unroll
    for (int i = 0; i < 7; i++) params[7ll * g + i] = p[i];
    info[3 * g] = inf2[0];
    info[3 * g + 1] = inf2[1];
    info[3 * g + 2] = cnt < 7 ? 1 : 0;
  }
}

// yhat[row] = predict7(params[model[g]], X[row]) for rows [lo[g], hi[g]) (`predict.py:43-44`)
__global__ void k_predict_segments(const double* __restrict__ X, const long long* __restrict__ lo,
                                   const long long* __restrict__ hi, const int32_t* __restrict__ model,
                                   const double* __restrict__ params, double* __restrict__ yhat) {
  const int g = blockIdx.x;
  double w[7];
  const int m = model ? model[g] : g;
#pragma unroll
  for (int i = 0; i < 7; i++) w[i] = params[7ll * m + i];
  for (long long row = lo[g] + threadIdx.x; row < hi[g]; row += blockDim.x) yhat[row] = predict7(w, X + row * 6);
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
// Dataset s is rows [off[s], off[s+1]) (or [off[s], end[s]) when end is given);
// blockIdx.y selects one of gridDim.y prediction vectors yhat + y_idx * yhat_stride,
// out[(s * gridDim.y + blockIdx.y) * 6 ..] = (mse, p25, p50, p75, p95, n).
__global__ void __launch_bounds__(kEvalThreads) k_eval(const double* __restrict__ yhat, const double* __restrict__ y,
                                                       const long long* __restrict__ off, double* __restrict__ out,
                                                       const long long* __restrict__ end = nullptr,
                                                       long long yhat_stride = 0, long long min_n = 0) {
  const int s = blockIdx.x;
  const long long a = off[s], n = (end ? end[s] : off[s + 1]) - a;
  if (n < min_n) return;  // done by k_eval_warp
  yhat += blockIdx.y * yhat_stride;
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
    double* o = out + 6ll * ((long long)s * gridDim.y + blockIdx.y);
    o[0] = n ? tot / (double)n : NAN;
    for (int q = 0; q < 4; q++) o[1 + q] = n ? key_f64(prefix[q]) : NAN;
    o[5] = (double)n;
  }
}

// EvalReports of small datasets (n <= kEvalWarpMax), one warp each: the
// relative errors are sorted in shared memory (bitonic, padded with +inf to a
// power of two) and the nearest-rank quantiles read off (`metrics.py:28-36`:
// sorted[ceil(p/100 n) - 1]); MSE by a warp sum.  Dataset s, vector k:
// rows [off[s], end[s]) of yhat + k * yhat_stride; out[(s * n_kinds + k) * 6].
constexpr int kEvalWarpMax = 1024, kEvalWarps = 4;
__global__ void __launch_bounds__(32 * kEvalWarps) k_eval_warp(const double* __restrict__ yhat,
                                                              const double* __restrict__ y,
                                                              const long long* __restrict__ off,
                                                              const long long* __restrict__ end, int n_seg,
                                                              int n_kinds, long long yhat_stride,
                                                              double* __restrict__ out) {
  __shared__ double v[kEvalWarps][kEvalWarpMax];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * kEvalWarps + wi;
  if (g >= (long long)n_seg * n_kinds) return;
  const int s = (int)(g / n_kinds), k = (int)(g % n_kinds);
  const long long a = off[s], n = end[s] - a;
  if (n > kEvalWarpMax) return;  // the block kernel's
  const double* yh = yhat + k * yhat_stride;
  double* buf = v[wi];
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  double sq = 0.0;
  for (int i = lane; i < np2; i += 32) {
    double rel = INFINITY;
    if (i < n) {
      const double d = yh[a + i] - y[a + i];
      sq = fma(d, d, sq);
      rel = fabs(d) / y[a + i];
    }
    buf[i] = rel;
  }
  sq = warp_sum(sq);
  __syncwarp();
  for (int kk = 2; kk <= np2; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < np2; i += 32) {
        const int p = i ^ j;
        if (p > i) {
          const double x = buf[i], z = buf[p];
          const bool up = (i & kk) == 0;
          if ((x > z) == up) {
            buf[i] = z;
            buf[p] = x;
          }
        }
      }
      __syncwarp();
    }
  if (lane < 6) {
    double r;
    if (n == 0) {
      r = lane == 5 ? 0.0 : NAN;
    } else if (lane == 0) {
      r = sq / (double)n;
    } else if (lane == 5) {
      r = (double)n;
    } else {
      const double pq = lane == 1 ? 25.0 : lane == 2 ? 50.0 : lane == 3 ? 75.0 : 95.0;
      long long rk = (long long)ceil((pq / 100.0) * (double)n);
      r = buf[(rk < 1 ? 1 : rk) - 1];
    }
    out[g * 6 + lane] = r;
  }
}

}  // namespace

long long cand_ws_elems(int E, long long ld) { return 3 * ld + 3LL * E * ld; }

template <int K>
static int launch_prep(const intf_table* t, int cap, double alpha, float* ws, cudaStream_t st) {
  const int E = t->n_rows;
  const long long sets = n_multisets(E, cap), ld = cand_ld(sets);
  const size_t smem = sizeof(unsigned long long) * (K + 1) * (E + K + 1);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_cand_prep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_cand_prep<K><<<dim3(ceil_div(ld, 128), ceil_div(E, kPrepOwn)), 128, smem, st>>>(t->solo_ms, t->thr, E, cap, sets,
                                                                                  ld, alpha, ws, ws + 3 * ld,
                                                                                  kPrepOwn);
  return launch_status("k_cand_prep");
}

static int launch_stream(const intf_table* t, int cap, const double* coefs, int n_dec, float* out, float* ws,
                         cudaStream_t st) {
  const int E = t->n_rows;
  const long long sets = n_multisets(E, cap), ld = cand_ld(sets);
  dim3 grid(ceil_div(ld / 4, kStreamThreads), E, ceil_div(n_dec, kStreamDec));
  k_cand_stream<<<grid, kStreamThreads, 0, st>>>(t->thr, E, ld, sets, coefs, n_dec, ws, ws + 3 * ld, out);
  return launch_status("k_cand_stream");
}

template <int K>
static int launch_step(const intf_table* t, int cap, double alpha, const double* coefs, int n_dec, float* out,
                       const float* ws_cur, float* ws_next, cudaStream_t st, unsigned long long* best = nullptr,
                       unsigned long long* best_next = nullptr) {
  const int E = t->n_rows;
  const long long sets = n_multisets(E, cap), ld = cand_ld(sets);
  const size_t smem = sizeof(unsigned long long) * (K + 1) * (E + K + 1);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_cand_step<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_cand_step<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const int po = kStepPrepOwn;
  const int px = (int)ceil_div(ld, 128), py = (int)ceil_div(E, po);
  const int sx = (int)ceil_div(ld / 4, kStreamThreads * (best ? kBestSpan : 1));
  const long long nblk = (ws_next ? (long long)px * py : 0) + (long long)sx * E * ceil_div(n_dec, kStreamDec);
  if (nblk > 0x7fffffffLL) return bad_input("intf_candidate_step: too many blocks");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nblk);
  cfg.blockDim = dim3(kStreamThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (best) {
    const long long n_best = 2ll * n_dec * E;
    cudaLaunchKernelEx(&cfg, k_cand_step<K, true>, t->solo_ms, t->thr, E, cap, sets, ld, alpha, coefs, n_dec, ws_cur,
                       ws_next, out, px, py, po, sx, best, best_next, n_best);
    return launch_status("k_cand_step<best>");
  }
  cudaLaunchKernelEx(&cfg, k_cand_step<K, false>, t->solo_ms, t->thr, E, cap, sets, ld, alpha, coefs, n_dec, ws_cur,
                     ws_next, out, px, py, po, sx, (unsigned long long*)nullptr, (unsigned long long*)nullptr, 0ll);
  return launch_status("k_cand_step");
}

// the device address of a pinned (page-locked, mapped) host buffer, or null
// for pageable memory (then the call copies).  Queried on every call (~1 us):
// a remembered address could have been freed and reused for pageable memory.
static unsigned long long* host_device_ptr(void* h) {
  cudaPointerAttributes a = {};
  void* d = nullptr;
  if (cudaPointerGetAttributes(&a, h) == cudaSuccess && a.type == cudaMemoryTypeHost) d = a.devicePointer;
  cudaGetLastError();  // (pageable memory: clear any error of the query)
  return reinterpret_cast<unsigned long long*>(d);
}

template <int K>
static int launch_step_host(const intf_table* t, int cap, double alpha, const double* h_coefs, int n_dec,
                            const float* ws_cur, float* ws_next, cudaStream_t st, unsigned long long* best,
                            unsigned* done, unsigned long long* host_best,
                            unsigned long long* flag = nullptr, unsigned long long seq = 0) {
  const int E = t->n_rows;
  const long long sets = n_multisets(E, cap), ld = cand_ld(sets);
  const size_t smem = sizeof(unsigned long long) * (K + 1) * (E + K + 1);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_cand_step_host<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int po = kStepPrepOwn;
  const int px = (int)ceil_div(ld, 128), py = (int)ceil_div(E, po);
  const int sx = (int)ceil_div(ld / 4, kStreamThreads * kBestSpan);
  const long long n_stream = (long long)sx * E * ceil_div(n_dec, kStreamDec);
  const long long nblk = (long long)px * py + n_stream;
  if (nblk > 0x7fffffffLL) return bad_input("intf_candidate_step: too many blocks");
  CandCoefs cp;
  memcpy(cp.c, h_coefs, sizeof(double) * n_dec * 2 * 7);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nblk);
  cfg.blockDim = dim3(kStreamThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const long long n_best = 2ll * n_dec * E;
  cudaLaunchKernelEx(&cfg, k_cand_step_host<K>, t->solo_ms, t->thr, E, cap, sets, ld, alpha, cp, n_dec, ws_cur,
                     ws_next, px, py, po, sx, best, n_best, done, (int)n_stream, host_best,
                     (volatile unsigned long long*)flag, seq);
  return launch_status("k_cand_step_host");
}

// phase: 1 = feature prep, 2 = forward stream, 3 = both (two-phase path only)
template <int K>
static int launch_candidates(const intf_table* t, int cap, double alpha, const double* coefs, int n_dec, float* out,
                             float* ws, long long ws_elems, cudaStream_t st, int phase = 3) {
  const int E = t->n_rows;
  const long long sets = n_multisets(E, cap), ld = cand_ld(sets);
  const size_t smem = sizeof(unsigned long long) * (K + 1) * (E + K + 1);
  if (smem > 200 * 1024) return bad_input("intf_predict_candidates: profile table too large for the binomial table");
  if (ws && ws_elems >= cand_ws_elems(E, ld)) {  // two-phase: prep (features) + stream (forward)
    int rc = (phase & 1) ? launch_prep<K>(t, cap, alpha, ws, st) : INTF_OK;
    if (rc || !(phase & 2)) return rc;
    return launch_stream(t, cap, coefs, n_dec, out, ws, st);
  }
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_candidates<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(ceil_div(ld / kGroup, kCandThreads), ceil_div(E, kOwnChunk), ceil_div(n_dec, kDecChunk));
  k_candidates<K><<<grid, kCandThreads, smem, st>>>(t->solo_ms, t->thr, E, cap, sets, ld, alpha, coefs, n_dec, out);
  return launch_status("k_candidates");
}

// tensor maps of the windowed refit's inputs over the n_full full windows:
// X as {16 doubles, window*6/16 groups, n_full windows} (128-byte swizzle),
// y as {window rows, n_full windows} (64-byte swizzle).  The encoder is the
// driver's, reached through the runtime (no libcuda link).
static int ols_window_maps(const double* X, const double* y, int window, long long n_full, CUtensorMap* mx, CUtensorMap* my) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      set_last_error("intf_ols_windows: cuTensorMapEncodeTiled unavailable");
      return INTF_E_CUDA;
    }
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dx[3] = {16, (cuuint64_t)(window * 6 / 16), (cuuint64_t)n_full};
  const cuuint64_t sx[2] = {128, (cuuint64_t)window * 48};
  const cuuint32_t bx[3] = {16, 3, 32}, ex[3] = {1, 1, 1};
  const cuuint64_t dy[2] = {(cuuint64_t)window, (cuuint64_t)n_full};
  const cuuint64_t sy[1] = {(cuuint64_t)window * 8};
  const cuuint32_t by[2] = {kWinTmaRows, 32}, ey[2] = {1, 1};
  const CUresult r1 = enc(mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dx, sx, bx, ex,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const CUresult r2 = enc(my, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(y), dy, sy, by, ey,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
    set_last_error("intf_ols_windows: tensor map encoding failed (%d, %d)", (int)r1, (int)r2);
    return INTF_E_CUDA;
  }
  return INTF_OK;
}

extern "C" {

int intf_candidate_count(int32_t n_rows, int32_t cap, int64_t* n_cand, int64_t* n_sets, int64_t* ld) {
  if (n_rows < 1 || cap < 1 || cap > kMaxPeers + 1 || !n_cand) return bad_input("intf_candidate_count: bad argument");
  const long long sets = n_multisets(n_rows, cap);
  *n_cand = (int64_t)n_rows * sets;
  if (n_sets) *n_sets = sets;
  if (ld) *ld = cand_ld(sets);
  return INTF_OK;
}

int intf_candidate_workspace(int32_t n_rows, int32_t cap, int64_t* ws_elems) {
  int64_t n_cand, n_sets, ld;
  int rc = intf_candidate_count(n_rows, cap, &n_cand, &n_sets, &ld);
  if (rc) return rc;
  if (!ws_elems) return bad_input("intf_candidate_workspace: null argument");
  *ws_elems = cand_ws_elems(n_rows, ld);
  return INTF_OK;
}

static int dispatch_candidates(const intf_table* table, int32_t cap, double alpha, const double* coefs, int32_t n_dec,
                               float* out, float* ws, int64_t ws_elems, void* stream, int phase) {
  cudaStream_t st = as_stream(stream);
  switch (cap - 1) {
    case 0: return launch_candidates<0>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
    case 1: return launch_candidates<1>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
    case 2: return launch_candidates<2>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
    case 3: return launch_candidates<3>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
    case 4: return launch_candidates<4>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
    case 5: return launch_candidates<5>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
    case 6: return launch_candidates<6>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
    default: return launch_candidates<7>(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, st, phase);
  }
}

int intf_predict_candidates(const intf_table* table, int32_t cap, double alpha, const double* coefs, int32_t n_dec,
                            float* out, float* ws, int64_t ws_elems, void* stream) {
  INTF_RANGE("intf_predict_candidates");
  if (!table || !coefs || !out || n_dec < 1 || cap < 1 || cap > kMaxPeers + 1 || table->n_rows < 1)
    return bad_input("intf_predict_candidates: bad argument (n_dec >= 1, 1 <= cap <= 8)");
  return dispatch_candidates(table, cap, alpha, coefs, n_dec, out, ws, ws_elems, stream, 3);
}

int intf_candidate_prepare(const intf_table* table, int32_t cap, double alpha, float* ws, int64_t ws_elems,
                           void* stream) {
  INTF_RANGE("intf_candidate_prepare");
  int64_t need = 0;
  if (!table || !ws || intf_candidate_workspace(table->n_rows, cap, &need) || ws_elems < need)
    return bad_input("intf_candidate_prepare: bad argument or workspace too small");
  return dispatch_candidates(table, cap, alpha, nullptr, 1, nullptr, ws, ws_elems, stream, 1);
}

int intf_predict_candidates_prepared(const intf_table* table, int32_t cap, const double* coefs, int32_t n_dec,
                                     float* out, const float* ws, int64_t ws_elems, void* stream) {
  INTF_RANGE("intf_predict_candidates_prepared");
  int64_t need = 0;
  if (!table || !coefs || !out || !ws || n_dec < 1 || intf_candidate_workspace(table->n_rows, cap, &need) ||
      ws_elems < need)
    return bad_input("intf_predict_candidates_prepared: bad argument or workspace too small");
  return launch_stream(table, cap, coefs, n_dec, out, const_cast<float*>(ws), as_stream(stream));
}

int intf_candidate_best_step(const intf_table* table, int32_t cap, double alpha, const double* coefs,
                             int32_t n_dec, uint64_t* best, uint64_t* best_next, const float* ws_cur, float* ws_next,
                             int64_t ws_elems, void* stream) {
  INTF_RANGE("intf_candidate_best_step");
  int64_t need = 0;
  if (!table || !coefs || !best || !ws_cur || !ws_next || n_dec < 1 || cap < 1 || cap > kMaxPeers + 1 ||
      intf_candidate_workspace(table->n_rows, cap, &need) || ws_elems < need || ws_next == ws_cur ||
      best_next == best)
    return bad_input("intf_candidate_best_step: bad argument or workspace too small");
  cudaStream_t st = as_stream(stream);
  unsigned long long *b = (unsigned long long*)best, *bn = (unsigned long long*)best_next;
  switch (cap - 1) {
    case 0: return launch_step<0>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
    case 1: return launch_step<1>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
    case 2: return launch_step<2>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
    case 3: return launch_step<3>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
    case 4: return launch_step<4>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
    case 5: return launch_step<5>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
    case 6: return launch_step<6>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
    default: return launch_step<7>(table, cap, alpha, coefs, n_dec, nullptr, ws_cur, ws_next, st, b, bn);
  }
}

int intf_candidate_step(const intf_table* table, int32_t cap, double alpha, const double* coefs, int32_t n_dec,
                        float* out, const float* ws_cur, float* ws_next, int64_t ws_elems, void* stream) {
  INTF_RANGE("intf_candidate_step");
  int64_t need = 0;
  if (!table || !coefs || !out || !ws_cur || n_dec < 1 || cap < 1 || cap > kMaxPeers + 1 ||
      intf_candidate_workspace(table->n_rows, cap, &need) || ws_elems < need || ws_next == ws_cur)
    return bad_input("intf_candidate_step: bad argument or workspace too small");
  cudaStream_t st = as_stream(stream);
  switch (cap - 1) {
    case 0: return launch_step<0>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
    case 1: return launch_step<1>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
    case 2: return launch_step<2>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
    case 3: return launch_step<3>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
    case 4: return launch_step<4>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
    case 5: return launch_step<5>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
    case 6: return launch_step<6>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
    default: return launch_step<7>(table, cap, alpha, coefs, n_dec, out, ws_cur, ws_next, st);
  }
}

int intf_predict_candidates_host(const intf_table* table, int32_t cap, double alpha, const double* h_coefs,
                                 int32_t n_dec, float* h_out, float* d_scratch, int64_t scratch_elems,
                                 void* stream) {
  INTF_RANGE("intf_predict_candidates_host");
  if (!table || !h_coefs || !h_out || !d_scratch) return bad_input("intf_predict_candidates_host: null argument");
  int64_t n_cand = 0, n_sets = 0, ld = 0, ws = 0;
  int rc = intf_candidate_count(table->n_rows, cap, &n_cand, &n_sets, &ld);
  if (rc) return rc;
  intf_candidate_workspace(table->n_rows, cap, &ws);
  const long long n_out = cand_out_elems(table->n_rows, ld, n_dec), n_coef = 2LL * n_dec * 2 * 7;
  if (scratch_elems < n_coef + n_out) return bad_input("intf_predict_candidates_host: scratch too small");
  cudaStream_t st = as_stream(stream);
  // scratch: [coefs as doubles][outputs][feature workspace, if it fits]
  double* d_coefs = reinterpret_cast<double*>(d_scratch);
  float* d_out = d_scratch + n_coef;
  float* d_ws = d_out + n_out;
  const long long ws_have = scratch_elems - n_coef - n_out;
  if (cudaMemcpyAsync(d_coefs, h_coefs, sizeof(double) * n_dec * 2 * 7, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return launch_status("copy coefs");
  rc = intf_predict_candidates(table, cap, alpha, d_coefs, n_dec, d_out, ws_have >= ws ? d_ws : nullptr, ws_have,
                               stream);
  if (rc) return rc;
  if (cudaMemcpyAsync(h_out, d_out, sizeof(float) * n_out, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return launch_status("copy predictions");
  return INTF_OK;
}

int intf_best_candidates_host(const intf_table* table, int32_t cap, double alpha, const double* h_coefs,
                              int32_t n_dec, uint64_t* h_best, float* d_scratch, int64_t scratch_elems,
                              void* stream) {
  INTF_RANGE("intf_best_candidates_host");
  if (!table || !h_coefs || !h_best || !d_scratch || n_dec < 1 || cap < 1 || cap > kMaxPeers + 1)
    return bad_input("intf_best_candidates_host: bad argument");
  int64_t ws = 0;
  intf_candidate_workspace(table->n_rows, cap, &ws);
  const long long n_coef = 2LL * n_dec * 2 * 7, n_best = 2LL * n_dec * table->n_rows;
  if (scratch_elems < n_coef + 2 * n_best + ws) return bad_input("intf_best_candidates_host: scratch too small");
  cudaStream_t st = as_stream(stream);
  // scratch: [coefs as doubles][best keys as u64][feature workspace]
  double* d_coefs = reinterpret_cast<double*>(d_scratch);
  unsigned long long* d_best = reinterpret_cast<unsigned long long*>(d_scratch + n_coef);
  float* d_ws = d_scratch + n_coef + 2 * n_best;
  if (cudaMemcpyAsync(d_coefs, h_coefs, sizeof(double) * n_dec * 2 * 7, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return launch_status("copy coefs");
  cudaMemsetAsync(d_best, 0xff, sizeof(unsigned long long) * n_best, st);
  int rc = intf_candidate_prepare(table, cap, alpha, d_ws, ws, stream);
  if (rc) return rc;
  switch (cap - 1) {
    case 0: rc = launch_step<0>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
    case 1: rc = launch_step<1>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
    case 2: rc = launch_step<2>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
    case 3: rc = launch_step<3>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
    case 4: rc = launch_step<4>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
    case 5: rc = launch_step<5>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
    case 6: rc = launch_step<6>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
    default: rc = launch_step<7>(table, cap, alpha, d_coefs, n_dec, nullptr, d_ws, nullptr, st, d_best); break;
  }
  if (rc) return rc;
  if (cudaMemcpyAsync(h_best, d_best, sizeof(unsigned long long) * n_best, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return launch_status("copy best candidates");
  return INTF_OK;
}

int intf_dispatch_sets(const intf_batch* bt, const intf_replay_buffers* buf, int32_t n_rows, int32_t cap_enum,
                       int32_t* dec_rank, int32_t* dec_own, void* stream) {
  INTF_RANGE("intf_dispatch_sets");
  if (!bt || !bt->scen || !bt->models || !buf || !buf->b_start || !buf->b_completion || !dec_rank || !dec_own ||
      cap_enum < 1 || cap_enum > kMaxPeers + 1 || buf->cap_max > cap_enum || n_rows < 1)
    return bad_input("intf_dispatch_sets: bad argument (the enumeration cap must cover every scenario's cap)");
  if (bt->n_scen <= 0) return INTF_OK;
  cudaMemsetAsync(dec_rank, 0xff, sizeof(int32_t) * (size_t)bt->req_slots, as_stream(stream));  // -1: no decision
  const int grid = bt->n_scen < 65535 ? bt->n_scen : 65535;
  k_dispatch_sets<<<grid, 128, 0, as_stream(stream)>>>(bt->scen, bt->n_scen, bt->models, *buf, n_rows, cap_enum,
                                                       dec_rank, dec_own);
  return launch_status("k_dispatch_sets");
}

int64_t intf_decision_features_elems(int32_t n_rows, int32_t cap) {
  return n_multisets(n_rows, cap) * 3ll * n_rows;
}

int intf_decision_features(const intf_table* table, int32_t cap, const float* ws, int64_t ws_elems, float* ft,
                           void* stream) {
  INTF_RANGE("intf_decision_features");
  int64_t need = 0;
  if (!table || !ws || !ft || intf_candidate_workspace(table->n_rows, cap, &need) || ws_elems < need)
    return bad_input("intf_decision_features: bad argument or workspace too small");
  const long long sets = n_multisets(table->n_rows, cap), ld = cand_ld(sets);
  const long long total = sets * 3ll * table->n_rows;
  k_decision_transpose<<<(unsigned)ceil_div(total, 256), 256, 0, as_stream(stream)>>>(ws + 3 * ld, table->n_rows, ld,
                                                                                    sets, ft);
  return launch_status("k_decision_transpose");
}

int intf_score_decisions_ft(const intf_table* table, int32_t cap, const double* coefs, const float* ws,
                            int64_t ws_elems, const float* ft, const int32_t* dec_rank, const int32_t* dec_own,
                            int64_t n, uint64_t* best, float* chosen, void* stream);

int intf_score_decisions(const intf_table* table, int32_t cap, const double* coefs, const float* ws, int64_t ws_elems,
                         const int32_t* dec_rank, const int32_t* dec_own, int64_t n, uint64_t* best, float* chosen,
                         void* stream) {
  INTF_RANGE("intf_score_decisions");
  return intf_score_decisions_ft(table, cap, coefs, ws, ws_elems, nullptr, dec_rank, dec_own, n, best, chosen, stream);
}

int intf_score_decisions_ft(const intf_table* table, int32_t cap, const double* coefs, const float* ws,
                            int64_t ws_elems, const float* ft, const int32_t* dec_rank, const int32_t* dec_own,
                            int64_t n, uint64_t* best, float* chosen, void* stream) {
  INTF_RANGE("intf_score_decisions_ft");
  int64_t need = 0;
  if (!table || !coefs || !ws || !dec_rank || !dec_own || !best || !chosen || n < 0 || table->n_rows > 64 ||
      intf_candidate_workspace(table->n_rows, cap, &need) || ws_elems < need)
    return bad_input("intf_score_decisions: bad argument, workspace too small or more than 64 profile rows");
  if (n == 0) return INTF_OK;
  const long long ld = cand_ld(n_multisets(table->n_rows, cap));
  if (ft) {  // decision-major features: a lane per decision
    const long long want = ceil_div(n, 128);
    k_score_decisions_lane<<<(unsigned)(want < 148 * 16 ? want : 148 * 16), 128, 0, as_stream(stream)>>>(
        table->thr, table->n_rows, ld, coefs, ws, ft, dec_rank, dec_own, (long long)n, (unsigned long long*)best,
        chosen);
    return launch_status("k_score_decisions_lane");
  }
  const long long want = ceil_div(n, 128);  // a warp per 32-slot group
  k_score_decisions<<<(unsigned)(want < 148 * 16 ? want : 148 * 16), 128, 0, as_stream(stream)>>>(
      table->thr, table->n_rows, ld, coefs, ws, ws + 3 * ld, dec_rank, dec_own, (long long)n,
      (unsigned long long*)best, chosen, ft);
  return launch_status("k_score_decisions");
}

static int best_host_pipelined(const intf_table* table, int32_t cap, double alpha, const double* h_coefs,
                               int32_t n_dec, uint64_t* h_best, float* d_scratch, int64_t scratch_elems,
                               int64_t* state, void* stream, unsigned long long* flag, unsigned long long seq,
                               bool* one_launch);

int intf_best_candidates_host_pipelined(const intf_table* table, int32_t cap, double alpha, const double* h_coefs,
                                        int32_t n_dec, uint64_t* h_best, float* d_scratch, int64_t scratch_elems,
                                        int64_t* state, void* stream) {
  INTF_RANGE("intf_best_candidates_host_pipelined");
  bool one = false;
  return best_host_pipelined(table, cap, alpha, h_coefs, n_dec, h_best, d_scratch, scratch_elems, state, stream,
                             nullptr, 0, &one);
}

// the per-thread pinned completion word of intf_best_candidates_host_sync
struct HostFlag {
  unsigned long long* h = nullptr;  // host view
  unsigned long long* d = nullptr;  // device view
  unsigned long long seq = 0;
  int dev = -1;
};
static HostFlag* host_flag() {
  static thread_local HostFlag f[16];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16) return nullptr;
  HostFlag& x = f[dev];
  if (!x.h) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    void* dp = nullptr;
    cudaHostGetDevicePointer(&dp, p, 0);
    x.h = reinterpret_cast<unsigned long long*>(p);
    x.d = reinterpret_cast<unsigned long long*>(dp);
    *x.h = 0;
    x.dev = dev;
  }
  return &x;
}

int intf_best_candidates_host_sync(const intf_table* table, int32_t cap, double alpha, const double* h_coefs,
                                   int32_t n_dec, uint64_t* h_best, float* d_scratch, int64_t scratch_elems,
                                   int64_t* state, void* stream) {
  INTF_RANGE("intf_best_candidates_host_sync");
  HostFlag* f = host_flag();
  const unsigned long long seq = f ? ++f->seq : 0;
  bool one = false;
  int rc = best_host_pipelined(table, cap, alpha, h_coefs, n_dec, h_best, d_scratch, scratch_elems, state, stream,
                               f ? f->d : nullptr, seq, &one);
  if (rc) return rc;
  if (!one || !f) {  // copy path: the stream's completion
    if (cudaStreamSynchronize(as_stream(stream)) != cudaSuccess) return launch_status("intf_best_candidates_host_sync");
    return INTF_OK;
  }
  // one-launch path: spin on the word the kernel's last block writes after the keys (a stream
  // synchronisation would add the completion's propagation); a stall falls back to it
  volatile unsigned long long* w = f->h;
  for (long long spin = 0; *w != seq; spin++) {
    if (spin > (1ll << 26)) {
      if (cudaStreamSynchronize(as_stream(stream)) != cudaSuccess)
        return launch_status("intf_best_candidates_host_sync");
      if (*w != seq) return bad_input("intf_best_candidates_host_sync: the kernel did not signal");
      break;
    }
  }
  return INTF_OK;
}

static int best_host_pipelined(const intf_table* table, int32_t cap, double alpha, const double* h_coefs,
                               int32_t n_dec, uint64_t* h_best, float* d_scratch, int64_t scratch_elems,
                               int64_t* state, void* stream, unsigned long long* flag, unsigned long long seq,
                               bool* one_launch) {
  if (!table || !h_coefs || !h_best || !d_scratch || !state || n_dec < 1 || cap < 1 || cap > kMaxPeers + 1)
    return bad_input("intf_best_candidates_host_pipelined: bad argument");
  int64_t ws = 0;
  intf_candidate_workspace(table->n_rows, cap, &ws);
  const long long n_coef = 2LL * n_dec * 2 * 7, n_best = 2LL * n_dec * table->n_rows;
  if (scratch_elems < n_coef + 2 * n_best + 2 * ws)
    return bad_input("intf_best_candidates_host_pipelined: scratch too small");
  cudaStream_t st = as_stream(stream);
  // scratch: [workspace 0][workspace 1][best keys as u64][coefs as doubles ... completion counter in
  // the last float], the workspaces and keys at offsets that do not depend on n_dec (consecutive
  // calls may score different numbers of decisions); *state counts calls: call k reads the
  // features call k-1 built into workspace k & 1 and builds call k+1's into the other
  float* d_ws[2] = {d_scratch, d_scratch + ws};
  unsigned long long* d_best = reinterpret_cast<unsigned long long*>(d_scratch + 2 * ws);
  double* d_coefs = reinterpret_cast<double*>(d_scratch + 2 * ws + 2 * n_best);
  int rc;
  // *state: bits 0-47 count the calls; bits 48-55 = the decisions whose keys
  // the one-launch path has armed (~0; each call re-arms its own range) and
  // whose completion counter is zero -- 0 after a copy-path call, which
  // overwrites them
  constexpr long long kCount = (1ll << 48) - 1;
  const long long k = *state & kCount;
  const int armed = (int)((*state >> 48) & 0xff);
  unsigned long long* h_dev = n_dec <= kHostDecMax ? host_device_ptr(h_best) : nullptr;
  if (h_dev) {  // one launch: coefficients as a parameter, keys written into the pinned buffer by the last block
    unsigned* done = reinterpret_cast<unsigned*>(d_scratch + scratch_elems - 1);  // (past the keys: n_coef >= 28)
    if (k == 0 && (rc = intf_candidate_prepare(table, cap, alpha, d_ws[0], ws, stream))) return rc;
    if (armed == 0) cudaMemsetAsync(done, 0, sizeof(unsigned), st);
    if (n_dec > armed) cudaMemsetAsync(d_best, 0xff, sizeof(unsigned long long) * n_best, st);
    switch (cap - 1) {
      case 0: rc = launch_step_host<0>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
      case 1: rc = launch_step_host<1>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
      case 2: rc = launch_step_host<2>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
      case 3: rc = launch_step_host<3>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
      case 4: rc = launch_step_host<4>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
      case 5: rc = launch_step_host<5>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
      case 6: rc = launch_step_host<6>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
      default: rc = launch_step_host<7>(table, cap, alpha, h_coefs, n_dec, d_ws[k & 1], d_ws[(k + 1) & 1], st, d_best, done, h_dev, flag, seq); break;
    }
    if (rc) return rc;
    *state = (k + 1) | ((long long)(n_dec > armed ? n_dec : armed) << 48);
    *one_launch = true;
    return INTF_OK;
  }
  if (cudaMemcpyAsync(d_coefs, h_coefs, sizeof(double) * n_dec * 2 * 7, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return launch_status("copy coefs");
  if (k == 0 && (rc = intf_candidate_prepare(table, cap, alpha, d_ws[0], ws, stream))) return rc;
  cudaMemsetAsync(d_best, 0xff, sizeof(unsigned long long) * n_best, st);
  float *cur = d_ws[k & 1], *nxt = d_ws[(k + 1) & 1];
  switch (cap - 1) {
    case 0: rc = launch_step<0>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
    case 1: rc = launch_step<1>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
    case 2: rc = launch_step<2>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
    case 3: rc = launch_step<3>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
    case 4: rc = launch_step<4>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
    case 5: rc = launch_step<5>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
    case 6: rc = launch_step<6>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
    default: rc = launch_step<7>(table, cap, alpha, d_coefs, n_dec, nullptr, cur, nxt, st, d_best); break;
  }
  if (rc) return rc;
  if (cudaMemcpyAsync(h_best, d_best, sizeof(unsigned long long) * n_best, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return launch_status("copy best candidates");
  *state = k + 1;
  return INTF_OK;
}

int intf_ols_stats(const double* X, const double* y, int64_t n, double* out, double* ws, void* stream) {
  INTF_RANGE("intf_ols_stats");
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
  INTF_RANGE("intf_ols_solve");
  if (!stats || !out_params) return bad_input("intf_ols_solve: null argument");
  k_ols_solve<<<1, 32, 0, as_stream(stream)>>>(stats, nullptr, out_params, out_info, out_Pinv);
  return launch_status("k_ols_solve");
}

int intf_ols_fit_rows(const double* X, const double* y, int64_t n, const double* stats, double* ws,
                      double* out_params, int32_t* out_info, double* out_Pinv, void* stream) {
  INTF_RANGE("intf_ols_fit_rows");
  if (!X || !y || !stats || !ws || !out_params || n < 0) return bad_input("intf_ols_fit_rows: bad argument");
  cudaStream_t st = as_stream(stream);
  const long long want = (n + 32ll * kQrThreads - 1) / (32ll * kQrThreads);  // >= 32 rows per thread
  const int nb = (int)(want < 1 ? 1 : want > kQrBlocks ? kQrBlocks : want);
  double* qr = ws + kQrBlocks * kQrPacked;
  k_ols_qr_rows<<<nb, kQrThreads, 0, st>>>(X, y, (long long)n, stats, ws);
  int rc = launch_status("k_ols_qr_rows");
  if (rc) return rc;
  k_ols_qr_final<<<1, kQrBlocks, 0, st>>>(stats, ws, nb, (double)n, qr);
  if ((rc = launch_status("k_ols_qr_final"))) return rc;
  k_ols_solve<<<1, 32, 0, st>>>(stats, qr, out_params, out_info, out_Pinv);
  return launch_status("k_ols_solve");
}

int intf_ols_windows(const double* X, const double* y, int64_t n, int32_t window, double* stats, double* params,
                     int32_t* info, void* stream) {
  INTF_RANGE("intf_ols_windows");
  if (!X || !y || !params || !info || n < 0 || window < 1)
    return bad_input("intf_ols_windows: bad argument");
  const long long n_win = (n + window - 1) / window;
  if (n_win == 0) return INTF_OK;
  cudaStream_t st = as_stream(stream);
  const long long n_full = n / window;
  if (window % kWinTmaRows == 0 && n_full >= 1 && n_full < (1ll << 31) && ((uintptr_t)X & 15) == 0 &&
      ((uintptr_t)y & 15) == 0) {
    CUtensorMap mx, my;
    int rc = ols_window_maps(X, y, window, n_full, &mx, &my);
    if (rc) return rc;
    int dev = 0;
    cudaGetDevice(&dev);
    static bool attr_set[64] = {};
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      cudaFuncSetAttribute(k_ols_windows_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kWinTmaSmem);
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
    const long long n_grp = (n_win + 31) / 32;
    const unsigned grid = (unsigned)(n_grp < 148 * kWinTmaPerSm ? n_grp : 148 * kWinTmaPerSm);
    k_ols_windows_tma<<<grid, 32, kWinTmaSmem, st>>>(mx, my, X, y, (long long)n, window, n_win, stats, params, info);
    return launch_status("k_ols_windows_tma");
  }
  if (window <= kFusedWindow) {
    k_ols_windows_fused<<<ceil_div(n_win, 128), 128, 0, st>>>(X, y, (long long)n, window, n_win, stats, params, info);
    return launch_status("k_ols_windows_fused");
  }
  if (!stats) return bad_input("intf_ols_windows: stats scratch needed for windows > 128 rows that are not a multiple of 8");
  k_ols_window_stats<<<ceil_div(n_win, kWinWarps), 32 * kWinWarps, 0, st>>>(X, y, (long long)n, window, n_win, stats);
  int rc = launch_status("k_ols_window_stats");
  if (rc) return rc;
  k_ols_window_solve<<<ceil_div(n_win, 128), 128, 0, st>>>(stats, X, y, n_win, (long long)n, window, params, info);
  return launch_status("k_ols_window_solve");
}

int intf_sgd_streams(const double* X, const double* y, const int64_t* off, int32_t n_streams, const double* eta,
                     double* params, double* pred, int32_t* status, void* stream) {
  INTF_RANGE("intf_sgd_streams");
  if (!X || !y || !off || !eta || !params || !pred || n_streams < 0) return bad_input("intf_sgd_streams: bad argument");
  if (n_streams == 0) return INTF_OK;
  k_sgd<<<ceil_div(n_streams, 64), 64, 0, as_stream(stream)>>>(X, y, (const long long*)off, n_streams, eta, params,
                                                               pred, status);
  return launch_status("k_sgd");
}

int intf_rls_streams(const double* X, const double* y, const int64_t* off, int32_t n_streams, const double* lam,
                     double* params, double* P, double* pred, int32_t* status, void* stream) {
  INTF_RANGE("intf_rls_streams");
  if (!X || !y || !off || !lam || !params || !P || !pred || n_streams < 0)
    return bad_input("intf_rls_streams: bad argument");
  if (n_streams == 0) return INTF_OK;
  k_rls_g8<<<ceil_div(n_streams, 128 / kRlsGroup), 128, 0, as_stream(stream)>>>(X, y, (const long long*)off, n_streams,
                                                                               lam, params, P, pred, status);
  return launch_status("k_rls_g8");
}

int64_t intf_scenario_eval_ws(int32_t n_scen, int64_t slot_stride) {
  // P0, lam, lo, hi, yhat; the designs' statistics, parameters and solve info
  return 49ll * n_scen + n_scen + 2ll * n_scen + 3ll * slot_stride + 112ll * n_scen + 14ll * n_scen + 2ll * n_scen;
}

int intf_scenario_eval(const intf_batch* bt, const intf_replay_buffers* buf, const double* X, int64_t slot_stride,
                       int32_t p_static, int32_t p_ewma, const double* y, double lam, double* ws, int64_t ws_elems,
                       double* params, double* report, int32_t* status, void* stream) {
  INTF_RANGE("intf_scenario_eval");
  if (!bt || !bt->scen || !buf || !buf->n_batches || !X || !y || !ws || !params || !report || !status ||
      p_static < 0 || p_ewma < 0 || !(lam > 0.0 && lam <= 1.0))
    return bad_input("intf_scenario_eval: bad argument");
  const int S = bt->n_scen;
  if (S <= 0) return INTF_OK;
  if (ws_elems < intf_scenario_eval_ws(S, slot_stride)) return bad_input("intf_scenario_eval: workspace too small");
  double* P0 = ws;
  double* lamv = P0 + 49ll * S;
  long long* lo = (long long*)(lamv + S);
  long long* hi = lo + S;
  double* yhat = (double*)(hi + S);
  double* stats = yhat + 3ll * slot_stride;  // [2S][56]
  double* par = stats + 112ll * S;          // [2S][7]
  int32_t* inf = (int32_t*)(par + 14ll * S);  // [2S][2]
  cudaStream_t st = as_stream(stream);
  k_scen_stats<<<ceil_div(2 * S, kScenFitWarps), 32 * kScenFitWarps, 0, st>>>(
      bt->scen, S, buf->n_batches, X, (long long)slot_stride, p_static, p_ewma, y, stats);
  int rc = launch_status("k_scen_stats");
  if (rc) return rc;
  k_scen_solve<<<ceil_div(2 * S, 128), 128, 0, st>>>(bt->scen, S, buf->n_batches, stats, par, inf);
  if ((rc = launch_status("k_scen_solve"))) return rc;
  k_scen_qr<<<ceil_div(S, kScenFitWarps), 32 * kScenFitWarps, 0, st>>>(
      bt->scen, S, buf->n_batches, X, (long long)slot_stride, p_static, p_ewma, y, stats, par, inf);
  if ((rc = launch_status("k_scen_qr"))) return rc;
  k_scen_finish<<<ceil_div(S, kScenFitWarps), 32 * kScenFitWarps, 0, st>>>(
      bt->scen, S, buf->n_batches, X, (long long)slot_stride, p_static, p_ewma, lam, stats, par, inf, params, P0,
      lamv, lo, hi, yhat, status);
  if ((rc = launch_status("k_scen_finish"))) return rc;
  // the adaptive tails: rls_update over EWMA[cut:], from the fine fit and P0 (params row 2 of each scenario)
  k_rls_g8<<<ceil_div(S, 128 / kRlsGroup), 128, 0, st>>>(X + (long long)p_ewma * slot_stride * 6, y, lo, S, lamv,
                                                          params + 14, P0, yhat + 2 * slot_stride, status + S, hi, 21);
  if ((rc = launch_status("k_rls_g8"))) return rc;
  k_eval_warp<<<ceil_div(3ll * S, kEvalWarps), 32 * kEvalWarps, 0, st>>>(yhat, y, lo, hi, S, 3, (long long)slot_stride,
                                                                        report);
  if ((rc = launch_status("k_eval_warp"))) return rc;
  // a test tail holds n - rint(0.75 n) <= n / 4 + 1 samples, n <= req_cap: if
  // every tail fits the warp kernel, the block kernel is not needed
  if ((long long)bt->max_req_cap / 4 + 1 <= kEvalWarpMax) return INTF_OK;
  k_eval<<<dim3(S, 3), kEvalThreads, 0, st>>>(yhat, y, lo, report, hi, (long long)slot_stride, kEvalWarpMax + 1);
  return launch_status("k_eval");
}

int intf_ols_fit_segments(const double* X, const double* y, const int64_t* lo, const int64_t* hi, int32_t n_seg,
                          double* params, int32_t* info, double* Pinv, void* stream) {
  INTF_RANGE("intf_ols_fit_segments");
  if (!X || !y || !lo || !hi || !params || !info || n_seg < 0) return bad_input("intf_ols_fit_segments: bad argument");
  if (n_seg == 0) return INTF_OK;
  k_fit_segments<<<ceil_div(n_seg, kScenFitWarps), 32 * kScenFitWarps, 0, as_stream(stream)>>>(
      X, y, (const long long*)lo, (const long long*)hi, n_seg, params, info, Pinv);
  return launch_status("k_fit_segments");
}

int intf_predict_segments(const double* X, const int64_t* lo, const int64_t* hi, const int32_t* model,
                          const double* params, int32_t n_seg, double* yhat, void* stream) {
  INTF_RANGE("intf_predict_segments");
  if (!X || !lo || !hi || !params || !yhat || n_seg < 0) return bad_input("intf_predict_segments: bad argument");
  if (n_seg == 0) return INTF_OK;
  k_predict_segments<<<n_seg, 128, 0, as_stream(stream)>>>(X, (const long long*)lo, (const long long*)hi, model,
                                                            params, yhat);
  return launch_status("k_predict_segments");
}

int intf_sgd_segments(const double* X, const double* y, const int64_t* lo, const int64_t* hi, int32_t n_seg,
                      const double* eta, double* params, double* pred, int32_t* status, void* stream) {
  INTF_RANGE("intf_sgd_segments");
  if (!X || !y || !lo || !hi || !eta || !params || !pred || n_seg < 0) return bad_input("intf_sgd_segments: bad argument");
  if (n_seg == 0) return INTF_OK;
  k_sgd<<<ceil_div(n_seg, 64), 64, 0, as_stream(stream)>>>(X, y, (const long long*)lo, n_seg, eta, params, pred, status,
                                                           (const long long*)hi);
  return launch_status("k_sgd");
}

int intf_rls_segments(const double* X, const double* y, const int64_t* lo, const int64_t* hi, int32_t n_seg,
                      const double* lam, double* params, double* P, double* pred, int32_t* status, void* stream) {
  INTF_RANGE("intf_rls_segments");
  if (!X || !y || !lo || !hi || !lam || !params || !P || !pred || n_seg < 0)
    return bad_input("intf_rls_segments: bad argument");
  if (n_seg == 0) return INTF_OK;
  k_rls_g8<<<ceil_div(n_seg, 128 / kRlsGroup), 128, 0, as_stream(stream)>>>(X, y, (const long long*)lo, n_seg, lam,
                                                                           params, P, pred, status,
                                                                           (const long long*)hi);
  return launch_status("k_rls_g8");
}

int intf_eval_segments(const double* yhat, const double* y, const int64_t* lo, const int64_t* hi, int32_t n_seg,
                       int64_t max_len, double* out, void* stream) {
  INTF_RANGE("intf_eval_segments");
  if (!yhat || !y || !lo || !hi || !out || n_seg < 0) return bad_input("intf_eval_segments: bad argument");
  if (n_seg == 0) return INTF_OK;
  cudaStream_t st = as_stream(stream);
  k_eval_warp<<<ceil_div(n_seg, kEvalWarps), 32 * kEvalWarps, 0, st>>>(yhat, y, (const long long*)lo,
                                                                      (const long long*)hi, n_seg, 1, 0, out);
  int rc = launch_status("k_eval_warp");
  if (rc || max_len <= kEvalWarpMax) return rc;
  k_eval<<<n_seg, kEvalThreads, 0, st>>>(yhat, y, (const long long*)lo, out, (const long long*)hi, 0,
                                         kEvalWarpMax + 1);
  return launch_status("k_eval");
}

int intf_eval_report(const double* yhat, const double* y, const int64_t* off, int32_t n_seg, double* out,
                     void* stream) {
  INTF_RANGE("intf_eval_report");
  if (!yhat || !y || !off || !out || n_seg < 0) return bad_input("intf_eval_report: bad argument");
  if (n_seg == 0) return INTF_OK;
  k_eval<<<n_seg, kEvalThreads, 0, as_stream(stream)>>>(yhat, y, (const long long*)off, out);
  return launch_status("k_eval");
}

}  // extern "C"
