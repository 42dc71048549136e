// replay.cu -- arrivals, scheduler replay, SLO accounting and per-outcome
// features for batches of scenarios (sm_100a).
//
// Layout in HBM (see include/intfsim_b200.h): scenarios are packed
// back-to-back; every per-request / per-batch array is indexed by
// req_off + i, per-model arrival lists by list_off + j, segments by
// seg_off + k.  All fp64 (the reference's arithmetic; bit-exactness needs
// the exact IEEE operations), compiled with -fmad=false.
#include <math.h>

#include "capi_common.h"
#include "replay_core.cuh"
#include "replay_warp.cuh"
#include "tma.cuh"

using namespace intf;

namespace {

#ifndef INTF_SCAN_SEQ
#define INTF_SCAN_SEQ 0  // 1: the one-thread add chain k_scan_gaps (A/B reference for the k_bin_* kernels)
#endif
#ifndef INTF_BIG_LIST
#define INTF_BIG_LIST 4096
#endif
constexpr int kBigList = INTF_BIG_LIST;  // model lists this long: parallel gaps + one-thread scan (long traces)
constexpr int kLongForm = INTF_LONG_LIST;  // model lists this long: chunked batch formation, time-bucket arrival merge
constexpr int kBigJobs = 1 << 15;  // scenarios this long: block-parallel job plan / verify
constexpr int kGapRun = 8;      // consecutive draws per thread in k_gen_gaps

// ---- K0a (long lists, e.g. one 10^6-request trace): every draw's gap of
// every long model stream in parallel (`workload.py:89-90`): draw d uses the
// PCG64 state after d+1 steps (LCG jump-ahead), u = (out >> 11) 2^-53,
// gap = max(-(1000/rate) log1p(-u), 1e-12), written into list_t as scratch.
__global__ void __launch_bounds__(256) k_gen_gaps(const intf_scenario* __restrict__ scen,
                                                  const intf_model* __restrict__ models, int n_models_total,
                                                  intf_replay_buffers B) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;
  if (g >= n_models_total) return;
  const intf_model& M = models[g];
  if (M.list_cap < kBigList || M.rate_rps == 0.0) return;
  const long long d0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kGapRun;
  if (d0 >= M.list_cap) return;
  const intf_scenario& S = scen[M.scen];
  uint32_t w[4];
  int nw = push_words(w, 0, S.seed);
  nw = push_words(w, nw, M.crc);
  const Pcg64 pg = pcg_seed_words(w, nw);
  const unsigned __int128 mult =
      ((unsigned __int128)0x2360ed051fc65da4ull << 64) | (unsigned __int128)0x4385df649fccf645ull;
  unsigned __int128 A, C;
  lcg_pow(mult, pg.inc, (unsigned long long)(d0 + 1), A, C);
  unsigned __int128 st = A * pg.state + C;
  const double neg_mean_gap = -(1000.0 / M.rate_rps);
  double* out = B.list_t + M.list_off;
#pragma unroll
  for (int r = 0; r < kGapRun; r++) {
    if (d0 + r >= M.list_cap) break;
    const double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
    const double gap = neg_mean_gap * glibc_log1p(-u);
    out[d0 + r] = gap > 1e-12 ? gap : 1e-12;
    st = mult * st + pg.inc;
  }
}

// ---- K0a' (long lists): every kScanChunk-th partial sum of t += gap
// (`workload.py:91`) goes into mb_t (free until formation) -- the k_bin_* kernels
// (below, the product) or the one-thread add chain k_scan_gaps (A/B
// reference, INTF_SCAN_SEQ=1); k_fill_gaps then redoes each chunk's adds --
// the same operations in the same order, so the same values -- in parallel
// and finds the horizon crossing.
constexpr int kScanChunk = 32;
#if INTF_SCAN_SEQ
constexpr int kScanStage = 512;  // doubles per bulk copy (4 KB)
constexpr int kScanStages = 4;   // copies in flight ahead of the add chain

// one block (one active thread) per long model: the gaps stream through
// shared memory by bulk copies kScanStages x 4 KB ahead of the add chain, so
// the chain runs at fp64 add latency; every 32nd partial sum goes to mb_t.
__global__ void __launch_bounds__(32) k_scan_gaps(const intf_scenario* __restrict__ scen,
                                                  const intf_model* __restrict__ models, int n_models_total,
                                                  intf_replay_buffers B) {
  __shared__ alignas(128) double buf[kScanStages][kScanStage];
  __shared__ alignas(8) uint64_t bar[kScanStages];
  const int g = blockIdx.x;
  if (g >= n_models_total || threadIdx.x != 0) return;
  const intf_model& M = models[g];
  if (M.list_cap < kBigList || M.rate_rps == 0.0) return;
  const double* lt = B.list_t + M.list_off;  // list_off is even: 16-byte aligned
  double* ends = B.mb_t + M.list_off;
  const int cap = M.list_cap, nch = (cap + kScanStage - 1) / kScanStage, n32 = cap / kScanChunk;
  const double horizon = scen[M.scen].duration_s * 1000.0;
  for (int i = 0; i < kScanStages; i++) mbar_init(&bar[i]);
  int issued = 0;
  auto issue = [&](int c) {
    const int lo = c * kScanStage, len = min(kScanStage, cap - lo);
    bulk_load(buf[c % kScanStages], lt + lo, (unsigned)((len + 1) & ~1) * 8u, &bar[c % kScanStages]);
    issued = c + 1;
  };
  for (int c = 0; c < kScanStages && c < nch; c++) issue(c);
  double t = 0.0;
  bool past = false;
  int c = 0;
  for (; c < nch && !past; c++) {
    mbar_wait(&bar[c % kScanStages], (unsigned)(c / kScanStages) & 1u);
    const double* sb = buf[c % kScanStages];
    const int lo = c * kScanStage, len = min(kScanStage, cap - lo);
    for (int k0 = 0; k0 < len; k0 += kScanChunk) {
      const int m = min(kScanChunk, len - k0);
      if (m == kScanChunk) {
#pragma unroll
        for (int k = 0; k < kScanChunk; k++) t = t + sb[k0 + k];
        ends[(lo + k0) / kScanChunk] = t;
        if (t >= horizon) {  // later 32-chunks lie past the horizon: k_fill_gaps skips them
          for (int e = (lo + k0) / kScanChunk + 1; e < n32; e++) ends[e] = INFINITY;
          past = true;
          break;
        }
      }  // a ragged tail (< 32) needs no end entry
    }
    if (!past && c + kScanStages < nch) issue(c + kScanStages);
  }
  // copies still in flight must land before the block (and its smem) exits
  for (int d = c; d < issued; d++) mbar_wait(&bar[d % kScanStages], (unsigned)(d / kScanStages) & 1u);
}

#endif  // INTF_SCAN_SEQ

// thread per (long model, chunk): rebuild the chunk's arrival times from the
// previous chunk's end; the chunk holding the horizon crossing sets n_list
__global__ void k_fill_gaps(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                            int n_models_total, intf_replay_buffers B) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;
  if (g >= n_models_total) return;
  const intf_model& M = models[g];
  if (M.list_cap < kBigList) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int cap = M.list_cap, nch = (cap + kScanChunk - 1) / kScanChunk;
  if (c >= nch) return;
  int n = -1;  // set by the thread that decides the count
  if (M.rate_rps == 0.0) {
    if (c == 0) n = 0;
  } else {
    const double horizon = scen[M.scen].duration_s * 1000.0;
    double* lt = B.list_t + M.list_off;
    const double* ends = B.mb_t + M.list_off;
    double t = c == 0 ? 0.0 : ends[c - 1];
    const int lo = c * kScanChunk, hi = lo + kScanChunk < cap ? lo + kScanChunk : cap;
    const bool below0 = t < horizon;  // (the ragged tail chunk also starts at ends[c - 1])
    for (int d = lo; d < hi; d++) {
      t = t + lt[d];
      lt[d] = t;
      if (n < 0 && below0 && t >= horizon) n = d;
    }
    if (n < 0 && hi == cap && t < horizon) n = cap + 1;  // still below the horizon: overflow
  }
  if (n >= 0) {
    if (n > M.list_cap) atomicOr(&B.status[M.scen], INTF_ST_OVERFLOW);
    B.n_list[g] = n;
    atomicAdd(&B.n_req[M.scen], n);
  }
}

// ---- K0a: one warp per deployed model generates its Poisson stream
// (warp-cooperative PCG64 jump-ahead, sequential cumulative sum).
constexpr int kGenWarps = 4;
__global__ void __launch_bounds__(32 * kGenWarps) k_gen_arrivals(const intf_scenario* __restrict__ scen,
                                                                 const intf_model* __restrict__ models,
                                                                 int n_models_total, intf_replay_buffers B) {
  __shared__ double gaps[kGenWarps][32];
  const int g = blockIdx.x * kGenWarps + (threadIdx.x >> 5);
  if (g >= n_models_total) return;
  const intf_model& M = models[g];
  if (M.list_cap >= kBigList) return;  // long lists: k_gen_gaps + k_scan_gaps
  const intf_scenario& S = scen[M.scen];
  const int n = gen_model_arrivals_warp(S, M, B.list_t + M.list_off, M.list_cap, gaps[threadIdx.x >> 5]);
  if ((threadIdx.x & 31) == 0) {
    if (n > M.list_cap) atomicOr(&B.status[M.scen], INTF_ST_OVERFLOW);
    B.n_list[g] = n;
    atomicAdd(&B.n_req[M.scen], n);
  }
}

// ---- K0b: merge per-model lists by (t, model_id) via rank = own index +
// elements of the other lists that precede it (binary search); one block per
// model list.  Writes the merged arrays and each element's request id.
__global__ void k_merge_arrivals(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                                 intf_replay_buffers B, int n_models) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;  // model lists beyond 65535 spill into grid.z
  if (g >= n_models) return;
  const intf_model M = models[g];
  const intf_scenario S = scen[M.scen];
  const int n = min(B.n_list[g], M.list_cap);
  if (B.status[M.scen] & INTF_ST_OVERFLOW) return;
  const double* lt = B.list_t + M.list_off;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double t = lt[j];
    int pos = j;
    for (int q = 0; q < S.n_models; q++) {
      const int gq = S.model_off + q;
      if (gq == g) continue;
      const intf_model& Q = models[gq];
      pos += count_before(B.list_t + Q.list_off, min(B.n_list[gq], Q.list_cap), t, Q.name_rank < M.name_rank);
    }
    if (pos < S.req_cap) {
      B.list_rid[M.list_off + j] = pos;
      B.arr_t[S.req_off + pos] = t;
      B.arr_model[S.req_off + pos] = g - S.model_off;
    }
  }
}

// The same merge by time buckets (long traces: a 10^6-request C4 trace spent
// 180 us in the 15 binary searches per element above).  Per scenario, in its
// share of form_ws (free until formation): nb = 2^k >= req_cap / 16 bucket
// counters and req_cap member slots.  Buckets are floor(t * nb / horizon),
// monotone in t; an element's merged position = its bucket's start + the
// members of its bucket that precede it under the same order as
// count_before ((t, name rank), then list index).  A bucket above 64 members
// (bursts) falls back to the binary searches for its elements.
constexpr int kArrBucketAvg = 16, kArrBucketMax = 64;
constexpr int kArrTile = 4096;  // buckets per scan tile (a block: 1024 threads x int4)
struct ArrBuckets {
  int32_t *cnt, *slot, *tile;  // local (per-tile) bucket offsets, members, tile offsets
  int nb;
  double scale;
  bool ok;
};
__device__ __forceinline__ ArrBuckets arr_buckets(const intf_scenario& S, const intf_model* __restrict__ models,
                                                  const intf_replay_buffers& B) {
  const intf_model& f = models[S.model_off];
  const intf_model& l = models[S.model_off + S.n_models - 1];
  const long long room = 3ll * ((long long)l.list_off + l.list_cap - f.list_off);
  int nb = 1;
  while ((long long)nb * kArrBucketAvg < S.req_cap) nb <<= 1;
  ArrBuckets A;
  A.cnt = B.form_ws + 3ll * f.list_off;
  A.slot = A.cnt + nb;
  A.tile = A.slot + S.req_cap;
  A.nb = nb;
  A.scale = (double)nb / (S.duration_s * 1000.0);
  A.ok = B.form_ws && S.duration_s > 0.0 && (long long)nb + S.req_cap + nb / kArrTile + 1 <= room &&
         S.n_models <= kMaxModels;
  return A;
}
// global offset of bucket b's current local counter
__device__ __forceinline__ int arr_at(const ArrBuckets& A, int b) { return A.cnt[b] + A.tile[b / kArrTile]; }
__device__ __forceinline__ int arr_bucket(const ArrBuckets& A, double t) {
  const double v = t * A.scale;
  return v < 0.0 ? 0 : (v >= (double)A.nb ? A.nb - 1 : (int)v);
}
// model list element (g, j) of a merge grid (as k_merge_arrivals)
struct ArrElem {
  int g, j, n;
  bool ok;
};
__device__ __forceinline__ ArrElem arr_elem(const intf_scenario* scen, const intf_model* models, int n_models,
                                            const intf_replay_buffers& B, int j) {
  ArrElem e;
  e.g = blockIdx.z * gridDim.y + blockIdx.y;
  e.j = j;
  e.ok = false;
  if (e.g >= n_models) return e;
  const intf_model& M = models[e.g];
  if (B.status[M.scen] & INTF_ST_OVERFLOW) return e;
  e.n = min(B.n_list[e.g], M.list_cap);
  e.ok = true;
  return e;
}
__global__ void __launch_bounds__(1024) k_arr_zero(const intf_scenario* __restrict__ scen,
                                                   const intf_model* __restrict__ models, intf_replay_buffers B) {
  const int s = blockIdx.y;  // (grid: tiles x scenarios)
  if (B.status[s] & INTF_ST_OVERFLOW) return;
  const ArrBuckets A = arr_buckets(scen[s], models, B);
  if (!A.ok) return;
  const int t0 = blockIdx.x * kArrTile;
  for (int b = t0 + threadIdx.x; b < min(A.nb, t0 + kArrTile); b += blockDim.x) A.cnt[b] = 0;
}
__global__ void k_arr_hist(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                           intf_replay_buffers B, int n_models) {
  const ArrElem e = arr_elem(scen, models, n_models, B, 0);
  if (!e.ok) return;
  const intf_model& M = models[e.g];
  const ArrBuckets A = arr_buckets(scen[M.scen], models, B);
  if (!A.ok) return;
  const double* lt = B.list_t + M.list_off;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < e.n; j += gridDim.x * blockDim.x)
    atomicAdd(&A.cnt[arr_bucket(A, lt[j])], 1);
}
// exclusive scan of the bucket counts: (1) per tile of kArrTile buckets, one
// block each (coalesced int4 loads), local offsets + the tile's total into
// tile[]; (2) one block per scenario scans the tile totals
__global__ void __launch_bounds__(1024) k_arr_scan_tiles(const intf_scenario* __restrict__ scen,
                                                         const intf_model* __restrict__ models,
                                                         intf_replay_buffers B) {
  __shared__ int wsum[32];
  const int s = blockIdx.y;  // (grid: tiles x scenarios)
  if (B.status[s] & INTF_ST_OVERFLOW) return;
  const ArrBuckets A = arr_buckets(scen[s], models, B);
  if (!A.ok) return;
  const int t0 = blockIdx.x * kArrTile;
  if (t0 >= A.nb) return;
  const int b0 = t0 + 4 * threadIdx.x;  // (4 consecutive counters per thread; form_ws offsets are only 4-byte aligned)
  int4 v = make_int4(0, 0, 0, 0);
  if (b0 < A.nb) v.x = A.cnt[b0];
  if (b0 + 1 < A.nb) v.y = A.cnt[b0 + 1];
  if (b0 + 2 < A.nb) v.z = A.cnt[b0 + 2];
  if (b0 + 3 < A.nb) v.w = A.cnt[b0 + 3];
  const int sum = v.x + v.y + v.z + v.w;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int u = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += y;
    }
    wsum[lane] = u;
  }
  __syncthreads();
  const int run = (w ? wsum[w - 1] : 0) + x - sum;
  if (b0 < A.nb) A.cnt[b0] = run;
  if (b0 + 1 < A.nb) A.cnt[b0 + 1] = run + v.x;
  if (b0 + 2 < A.nb) A.cnt[b0 + 2] = run + v.x + v.y;
  if (b0 + 3 < A.nb) A.cnt[b0 + 3] = run + v.x + v.y + v.z;
  if (threadIdx.x == blockDim.x - 1) A.tile[blockIdx.x] = wsum[31];  // the tile's total (before the scan below)
}
__global__ void k_arr_scan_top(const intf_scenario* __restrict__ scen, int n_scen,
                               const intf_model* __restrict__ models, intf_replay_buffers B) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_scen; s += gridDim.x * blockDim.x) {
    if (B.status[s] & INTF_ST_OVERFLOW) continue;
    const ArrBuckets A = arr_buckets(scen[s], models, B);
    if (!A.ok) continue;
    int run = 0;
    for (int k = 0; k * kArrTile < A.nb; k++) {
      const int c = A.tile[k];
      A.tile[k] = run;
      run += c;
    }
  }
}
__global__ void k_arr_scatter(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                              intf_replay_buffers B, int n_models) {
  const ArrElem e = arr_elem(scen, models, n_models, B, 0);
  if (!e.ok) return;
  const intf_model& M = models[e.g];
  const intf_scenario& S = scen[M.scen];
  const ArrBuckets A = arr_buckets(S, models, B);
  if (!A.ok) return;
  const double* lt = B.list_t + M.list_off;
  const int q = e.g - S.model_off;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < e.n; j += gridDim.x * blockDim.x) {
    const int b = arr_bucket(A, lt[j]);
    const int p = atomicAdd(&A.cnt[b], 1) + A.tile[b / kArrTile];  // (afterwards cnt[b] = the bucket's local end)
    if (p < S.req_cap) A.slot[p] = (q << 24) | j;
  }
}
__global__ void k_arr_place(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                            intf_replay_buffers B, int n_models) {
  const ArrElem e = arr_elem(scen, models, n_models, B, 0);
  if (!e.ok) return;
  const intf_model& M = models[e.g];
  const intf_scenario& S = scen[M.scen];
  const ArrBuckets A = arr_buckets(S, models, B);
  const double* lt = B.list_t + M.list_off;
  const int q = e.g - S.model_off;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < e.n; j += gridDim.x * blockDim.x) {
    const double t = lt[j];
    int pos = -1;
    if (A.ok) {
      const int b = arr_bucket(A, t);
      const int lo = b ? arr_at(A, b - 1) : 0, hi = arr_at(A, b);
      if (hi - lo <= kArrBucketMax) {
        int r = 0;
        for (int k = lo; k < hi; k++) {
          const int v = A.slot[k], q2 = v >> 24, j2 = v & 0xffffff;
          if (q2 == q) {
            r += j2 < j ? 1 : 0;
          } else {
            const intf_model& Q = models[S.model_off + q2];
            const double t2 = B.list_t[Q.list_off + j2];
            r += (t2 < t || (t2 == t && Q.name_rank < M.name_rank)) ? 1 : 0;
          }
        }
        pos = lo + r;
      }
    }
    if (pos < 0) {  // (no buckets for this scenario, or a burst bucket)
      pos = j;
      for (int q2 = 0; q2 < S.n_models; q2++) {
        if (q2 == q) continue;
        const intf_model& Q = models[S.model_off + q2];
        pos += count_before(B.list_t + Q.list_off, min(B.n_list[S.model_off + q2], Q.list_cap), t,
                            Q.name_rank < M.name_rank);
      }
    }
    if (pos < S.req_cap) {
      B.list_rid[M.list_off + j] = pos;
      B.arr_t[S.req_off + pos] = t;
      B.arr_model[S.req_off + pos] = q;
    }
  }
}

// The batch rank-merge of long traces by the same time buckets (over the
// formation times; window expiries past the horizon fall in the last
// bucket): a batch's global id = its bucket's start + the batches of its
// bucket preceding it in (t, kind, key) heap order (`simcore.py:122`), or,
// for the same model, in list order.  A bucket above 64 batches falls back to
// the binary searches of k_merge_batches.
__global__ void k_bat_hist(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                           intf_replay_buffers B, int n_models) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;
  if (g >= n_models) return;
  const intf_model& M = models[g];
  if (B.status[M.scen] & INTF_ST_OVERFLOW) return;
  const ArrBuckets A = arr_buckets(scen[M.scen], models, B);
  if (!A.ok) return;
  const int n = B.n_mb[g];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    atomicAdd(&A.cnt[arr_bucket(A, B.mb_t[M.list_off + j])], 1);
}
__global__ void k_bat_scatter(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                              intf_replay_buffers B, int n_models) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;
  if (g >= n_models) return;
  const intf_model& M = models[g];
  const intf_scenario& S = scen[M.scen];
  if (B.status[M.scen] & INTF_ST_OVERFLOW) return;
  const ArrBuckets A = arr_buckets(S, models, B);
  if (!A.ok) return;
  const int n = B.n_mb[g], q = g - S.model_off;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(&B.n_batches[M.scen], n);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int b = arr_bucket(A, B.mb_t[M.list_off + j]);
    const int p = atomicAdd(&A.cnt[b], 1) + A.tile[b / kArrTile];
    if (p < S.req_cap) A.slot[p] = (q << 24) | j;
  }
}
__global__ void k_bat_place(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                            intf_replay_buffers B, int n_models) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;
  if (g >= n_models) return;
  const intf_model& M = models[g];
  const intf_scenario& S = scen[M.scen];
  if (B.status[M.scen] & INTF_ST_OVERFLOW) return;
  const ArrBuckets A = arr_buckets(S, models, B);
  const int n = B.n_mb[g], q = g - S.model_off;
  if (!A.ok && blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(&B.n_batches[M.scen], n);  // (else: scatter's)
  const int ro = S.req_off;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double t = B.mb_t[M.list_off + j];
    const int4 info = reinterpret_cast<const int4*>(B.mb_info)[M.list_off + j];
    const int kind = info.x, cnt = info.z, head = info.w;
    const uint32_t key = (uint32_t)info.y;
    int rank = -1;
    if (A.ok) {
      const int b = arr_bucket(A, t);
      const int lo = b ? arr_at(A, b - 1) : 0, hi = arr_at(A, b);
      if (hi - lo <= kArrBucketMax) {
        int r = 0;
        for (int k = lo; k < hi; k++) {
          const int v = A.slot[k], q2 = v >> 24, j2 = v & 0xffffff;
          if (q2 == q) {
            r += j2 < j ? 1 : 0;
          } else {
            const intf_model& Q = models[S.model_off + q2];
            const int4 i2 = reinterpret_cast<const int4*>(B.mb_info)[Q.list_off + j2];
            r += form_key_less(B.mb_t[Q.list_off + j2], i2.x, (uint32_t)i2.y, t, kind, key) ? 1 : 0;
          }
        }
        rank = lo + r;
      }
    }
    if (rank < 0) {  // (no buckets, or a burst bucket)
      rank = j;
      for (int q2 = 0; q2 < S.n_models; q2++) {
        const int gq = S.model_off + q2;
        if (gq == g) continue;
        const intf_model& Q = models[gq];
        rank += count_form_before(B.mb_t + Q.list_off, B.mb_info + 4ll * Q.list_off, B.n_mb[gq], t, kind, key);
      }
    }
    B.b_model[ro + rank] = q;
    B.b_size[ro + rank] = cnt;
    B.b_formed[ro + rank] = t;
    const int32_t* lrid = B.list_rid + M.list_off;
    for (int k = 0; k < cnt; k++) B.r_batch[ro + lrid[head + k]] = rank;
  }
}

// The same merge with one block per SCENARIO for sweeps of many short
// scenarios: the scenario's model lists are staged in shared memory once and
// every element's rank is a binary search there (the per-model-list blocks
// above re-read the other lists from L2 on every search step).  Scenarios
// whose lists do not fit (kMergeSmem elements) take the global searches.
constexpr int kMergeSmem = 4096;
__global__ void __launch_bounds__(256) k_merge_arrivals_scen(const intf_scenario* __restrict__ scen, int n_scen,
                                                              const intf_model* __restrict__ models,
                                                              intf_replay_buffers B) {
  __shared__ double sl[kMergeSmem];
  __shared__ int soff[kMaxModels + 1];
  for (int s = blockIdx.x; s < n_scen; s += gridDim.x) {
    const intf_scenario S = scen[s];
    if (B.status[s] & INTF_ST_OVERFLOW) continue;
    if (threadIdx.x == 0) {
      int o = 0;
      for (int q = 0; q < S.n_models; q++) {
        soff[q] = o;
        const intf_model& Q = models[S.model_off + q];
        o += min(B.n_list[S.model_off + q], Q.list_cap);
      }
      soff[S.n_models] = o;
    }
    __syncthreads();
    const int total = soff[S.n_models];
    const bool fits = total <= kMergeSmem;
    if (fits) {
      for (int q = 0; q < S.n_models; q++) {
        const double* lt = B.list_t + models[S.model_off + q].list_off;
        for (int j = threadIdx.x; j < soff[q + 1] - soff[q]; j += blockDim.x) sl[soff[q] + j] = lt[j];
      }
    }
    __syncthreads();
    for (int q = 0; q < S.n_models; q++) {
      const int g = S.model_off + q;
      const intf_model& M = models[g];
      const int n = soff[q + 1] - soff[q];
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double t = fits ? sl[soff[q] + j] : B.list_t[M.list_off + j];
        int pos = j;
        for (int r = 0; r < S.n_models; r++) {
          if (r == q) continue;
          const intf_model& Q = models[S.model_off + r];
          const int nq = soff[r + 1] - soff[r];
          pos += fits ? count_before(sl + soff[r], nq, t, Q.name_rank < M.name_rank)
                      : count_before(B.list_t + Q.list_off, nq, t, Q.name_rank < M.name_rank);
        }
        if (pos < S.req_cap) {
          B.list_rid[M.list_off + j] = pos;
          B.arr_t[S.req_off + pos] = t;
          B.arr_model[S.req_off + pos] = q;
        }
      }
    }
    __syncthreads();
  }
}

// ---- split caller-supplied merged arrivals into per-model lists (serial
// per scenario; only for externally supplied traces).
__global__ void k_split_arrivals(const intf_scenario* __restrict__ scen, int n_scen,
                                 const intf_model* __restrict__ models, intf_replay_buffers B) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_scen) return;
  const intf_scenario S = scen[s];
  int cnt[kMaxModels];
  for (int m = 0; m < S.n_models && m < kMaxModels; m++) cnt[m] = 0;
  const int n = B.n_req[s];
  int st = 0;
  for (int i = 0; i < n; i++) {
    const int m = B.arr_model[S.req_off + i];
    const intf_model& M = models[S.model_off + m];
    if (cnt[m] < M.list_cap) {
      B.list_t[M.list_off + cnt[m]] = B.arr_t[S.req_off + i];
      B.list_rid[M.list_off + cnt[m]] = i;
    } else {
      st |= INTF_ST_OVERFLOW;
    }
    cnt[m]++;
  }
  for (int m = 0; m < S.n_models && m < kMaxModels; m++) B.n_list[S.model_off + m] = cnt[m];
  B.status[s] |= st;
}

// ---- K1 (per model): formation of every deployed model's batch list, one
// warp per model; then a block per model ranks its batches among all the
// scenario's batches by the heap key (time, kind, key) -> global batch ids.
constexpr int kFormModelWarps = 4;
__global__ void __launch_bounds__(32 * kFormModelWarps) k_form_models(const intf_scenario* __restrict__ scen,
                                                                      const intf_model* __restrict__ models,
                                                                      int n_models_total, intf_replay_buffers B) {
  const int g = blockIdx.x * kFormModelWarps + (threadIdx.x >> 5);
  if (g >= n_models_total) return;
  const intf_model& M = models[g];
  if (M.list_cap >= kLongForm) return;  // long lists: k_form_nxt .. k_form_emit
  const intf_scenario& S = scen[M.scen];
  const bool bad = (B.status[M.scen] & INTF_ST_OVERFLOW) || S.cap > B.cap_max || S.cap > kMaxCap || S.cap < 1 ||
                   S.max_bs < 1 || S.n_models > kMaxModels;
  if (bad) {
    if ((threadIdx.x & 31) == 0) B.n_mb[g] = 0;
    return;
  }
  form_model_warp(S, M, min(B.n_list[g], M.list_cap), B, g);
}

// ---- K1a' (long model lists, e.g. a 10^6-request trace): the batch starts
// of one model are the orbit h_0 = 0, h_{i+1} = nxt(h_i) = h_i + cnt(h_i),
// cnt(h) = next_formation's member count from head h (`batcher.py:44-85`),
// which is a pure function of h.  nxt for every h is computed in parallel,
// then the orbit by pointer doubling (J_{k+1} = J_k o J_k; path entries
// [2^k, 2^{k+1}) = J_k of entries [0, 2^k)), so the serial walk over the
// batches disappears.  Same batches, same events as form_model_warp.
__device__ __forceinline__ int form_cnt(const double* lt, int n, int h, double window, int max_bs) {
  const double D = lt[h] + window;  // arm_window at the first arrival (`batcher.py:66-68`)
  int lo = h + 1, hi = min(n, h + max_bs);  // first j in [h+1, hi) with lt[j] >= D, else hi
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (lt[mid] < D) lo = mid + 1;
    else hi = mid;
  }
  return lo - h;
}

struct LongModel {  // model g of a long-list launch (grid.y/z = model, grid.x = list chunk;
  int g, n, i;       // or a flat grid over bt->long_blocks: block b = (model, chunk) pair b)
  bool ok;
};
__device__ __forceinline__ LongModel long_model(const intf_scenario* scen, const intf_model* models, int n_models,
                                                const intf_replay_buffers& B, const int32_t* blk = nullptr) {
  LongModel r;
  r.g = blk ? blk[2 * blockIdx.x] : blockIdx.z * gridDim.y + blockIdx.y;
  r.ok = false;
  if (r.g >= n_models) return r;
  const intf_model& M = models[r.g];
  const intf_scenario& S = scen[M.scen];
  if (M.list_cap < kLongForm) return r;
  if ((B.status[M.scen] & INTF_ST_OVERFLOW) || S.cap > B.cap_max || S.cap > kMaxCap || S.cap < 1 || S.max_bs < 1 ||
      S.n_models > kMaxModels)
    return r;
  r.n = min(B.n_list[r.g], M.list_cap);
  r.i = (blk ? blk[2 * blockIdx.x + 1] : blockIdx.x) * blockDim.x + threadIdx.x;
  r.ok = true;
  return r;
}

// nxt(i) = i + cnt(i): the head after a batch starting at element i
__global__ void k_form_nxt(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                           int n_models, intf_replay_buffers B, const int32_t* blk) {
  const LongModel L = long_model(scen, models, n_models, B, blk);
  if (!L.ok || L.i >= L.n) return;
  const intf_model& M = models[L.g];
  const intf_scenario& S = scen[M.scen];
  int32_t* ws = B.form_ws + 3ll * M.list_off;  // [nxt | exit | count], list_cap each
  ws[L.i] = L.i + form_cnt(B.list_t + M.list_off, L.n, L.i, S.window_ms, S.max_bs);
}

// Long lists, chunked: the heads are the orbit of 0 under nxt(i) = i +
// cnt(i).  (1) k_form_chunks, a block per 2,048-element chunk: for EVERY
// element i of the chunk, the first head at or past the chunk's end reached
// from i and the heads visited on the way (pointer doubling in shared
// memory, 11 rounds) -> exit[i], count[i].  (2) k_form_compose, a thread per
// model: the walk from 0 jumps chunk to chunk through exit[] (one step per
// chunk), leaving each chunk's entry head and its first batch index in the
// chunk's first slot.  (3) k_form_emit_chunks, a block per chunk: one lane
// walks from the entry collecting the chunk's heads in shared memory, then the
// block writes their batch records (what form_model_warp writes).  Four
// launches instead of two per doubling level.
constexpr int kFormChunk = 2048;
constexpr int kFormChunkThreads = 256;
struct FormChunk {
  int g, c, n, lo, hi;  // model, chunk, list length, chunk [lo, hi)
  bool ok;
};
__device__ __forceinline__ FormChunk form_chunk(const intf_scenario* scen, const intf_model* models, int n_models,
                                                const intf_replay_buffers& B) {
  FormChunk f;
  f.g = blockIdx.z * gridDim.y + blockIdx.y;
  f.c = blockIdx.x;
  f.ok = false;
  if (f.g >= n_models) return f;
  const intf_model& M = models[f.g];
  const intf_scenario& S = scen[M.scen];
  if (M.list_cap < kLongForm) return f;
  if ((B.status[M.scen] & INTF_ST_OVERFLOW) || S.cap > B.cap_max || S.cap > kMaxCap || S.cap < 1 || S.max_bs < 1 ||
      S.n_models > kMaxModels)
    return f;
  f.n = min(B.n_list[f.g], M.list_cap);
  f.lo = f.c * kFormChunk;
  f.hi = min(f.n, f.lo + kFormChunk);
  f.ok = f.lo < f.n;
  return f;
}

__global__ void __launch_bounds__(kFormChunkThreads) k_form_chunks(const intf_scenario* __restrict__ scen,
                                                                   const intf_model* __restrict__ models,
                                                                   int n_models, intf_replay_buffers B) {
  const FormChunk f = form_chunk(scen, models, n_models, B);
  if (!f.ok) return;
  const intf_model& M = models[f.g];
  const int32_t* nxt = B.form_ws + 3ll * M.list_off;
  int32_t* exitv = B.form_ws + 3ll * M.list_off + M.list_cap;
  int32_t* count = B.form_ws + 3ll * M.list_off + 2ll * M.list_cap;
  __shared__ int32_t E[kFormChunk], K[kFormChunk];
  const int len = f.hi - f.lo;
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    E[j] = nxt[f.lo + j];
    K[j] = 1;
  }
  __syncthreads();
  // E[j]: the element reached; inside the chunk it is a head still to be followed
  for (int r = 0; (1 << r) < len; r++) {
    int e2[kFormChunk / kFormChunkThreads], k2[kFormChunk / kFormChunkThreads];
#pragma unroll
    for (int u = 0; u < kFormChunk / kFormChunkThreads; u++) {
      const int j = u * kFormChunkThreads + threadIdx.x;
      e2[u] = -1;
      if (j < len) {
        const int e = E[j];
        if (e < f.hi) {  // (e > lo + j >= lo: inside the chunk)
          e2[u] = E[e - f.lo];
          k2[u] = K[j] + K[e - f.lo];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kFormChunk / kFormChunkThreads; u++) {
      const int j = u * kFormChunkThreads + threadIdx.x;
      if (e2[u] >= 0) {
        E[j] = e2[u];
        K[j] = k2[u];
      }
    }
    __syncthreads();
  }
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    exitv[f.lo + j] = E[j];
    count[f.lo + j] = K[j];
  }
}

// per long model: chunk entries and first batch indices into each chunk's
// first exit / count slot (-1: no head in the chunk); n_mb = the batches
__global__ void k_form_compose(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                               int n_models, intf_replay_buffers B) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_models) return;
  const intf_model& M = models[g];
  if (M.list_cap < kLongForm) return;
  const intf_scenario& S = scen[M.scen];
  if ((B.status[M.scen] & INTF_ST_OVERFLOW) || S.cap > B.cap_max || S.cap > kMaxCap || S.cap < 1 || S.max_bs < 1 ||
      S.n_models > kMaxModels) {
    B.n_mb[g] = 0;  // long models of bad scenarios form nothing
    return;
  }
  const int n = min(B.n_list[g], M.list_cap);
  int32_t* exitv = B.form_ws + 3ll * M.list_off + M.list_cap;
  int32_t* count = B.form_ws + 3ll * M.list_off + 2ll * M.list_cap;
  int h = 0, base = 0;
  for (int c = 0; c * kFormChunk < n; c++) {
    const int lo = c * kFormChunk;
    if (h >= lo + kFormChunk || h >= n) {  // a batch skipped this whole chunk (or the orbit ended)
      exitv[lo] = -1;
      continue;
    }
    const int e = exitv[h], k = count[h];
    exitv[lo] = h;
    count[lo] = base;
    base += k;
    h = e;
  }
  B.n_mb[g] = base;
}

__global__ void __launch_bounds__(kFormChunkThreads) k_form_emit_chunks(const intf_scenario* __restrict__ scen,
                                                                        const intf_model* __restrict__ models,
                                                                        int n_models, intf_replay_buffers B) {
  const FormChunk f = form_chunk(scen, models, n_models, B);
  if (!f.ok) return;
  const intf_model& M = models[f.g];
  const intf_scenario& S = scen[M.scen];
  const int32_t* nxt = B.form_ws + 3ll * M.list_off;
  const int entry = B.form_ws[3ll * M.list_off + M.list_cap + f.lo];
  const int base = B.form_ws[3ll * M.list_off + 2ll * M.list_cap + f.lo];
  if (entry < 0) return;
  __shared__ int32_t nx[kFormChunk], heads[kFormChunk];
  __shared__ int n_heads;
  const int len = f.hi - f.lo;
  for (int j = threadIdx.x; j < len; j += blockDim.x) nx[j] = nxt[f.lo + j];
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0;
    for (int h = entry; h < f.hi; h = nx[h - f.lo]) heads[k++] = h;
    n_heads = k;
  }
  __syncthreads();
  const double* lt = B.list_t + M.list_off;
  const int32_t* lrid = B.list_rid + M.list_off;
  for (int j = threadIdx.x; j < n_heads; j += blockDim.x) {
    const int h = heads[j];
    const int cnt = nx[h - f.lo] - h;
    double t;
    int kind;
    uint32_t key;
    if (cnt == S.max_bs) {  // early emit at max_batch_size (`batcher.py:70-71`)
      t = lt[h + cnt - 1];
      kind = KIND_ARRIVAL;
      key = (uint32_t)lrid[h + cnt - 1];
    } else {  // window expiry (`batcher.py:74-85`)
      t = lt[h] + S.window_ms;
      kind = KIND_WINDOW;
      key = M.crc;
    }
    const int i = base + j;
    B.mb_t[M.list_off + i] = t;
    reinterpret_cast<int4*>(B.mb_info)[M.list_off + i] = make_int4(kind, (int32_t)key, cnt, h);
  }
}

__global__ void k_merge_batches(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                                intf_replay_buffers B, int n_models) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;
  if (g >= n_models) return;
  const intf_model& M = models[g];
  const intf_scenario& S = scen[M.scen];
  const int n = B.n_mb[g];
  const int mloc = g - S.model_off;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(&B.n_batches[M.scen], n);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double t = B.mb_t[M.list_off + j];
    const int32_t* info = B.mb_info + 4ll * (M.list_off + j);
    const int kind = info[0], cnt = info[2], head = info[3];
    const uint32_t key = (uint32_t)info[1];
    int rank = j;
    for (int q = 0; q < S.n_models; q++) {
      const int gq = S.model_off + q;
      if (gq == g) continue;
      const intf_model& Q = models[gq];
      rank += count_form_before(B.mb_t + Q.list_off, B.mb_info + 4ll * Q.list_off, B.n_mb[gq], t, kind, key);
    }
    const int ro = S.req_off;
    B.b_model[ro + rank] = mloc;
    B.b_size[ro + rank] = cnt;
    B.b_formed[ro + rank] = t;
    const int32_t* lrid = B.list_rid + M.list_off;
    for (int k = 0; k < cnt; k++) B.r_batch[ro + lrid[head + k]] = rank;
  }
}

// The same merge with one warp per model (sweeps of short lists: a C5 model
// forms ~100 batches, so k_merge_batches' 256-thread chunks were mostly idle
// block prologues)
__device__ __forceinline__ void merge_batch(const intf_scenario& S, const intf_model* __restrict__ models,
                                            const intf_replay_buffers& B, int g, int mloc, int j) {
  const intf_model& M = models[g];
  const double t = B.mb_t[M.list_off + j];
  const int4 info = reinterpret_cast<const int4*>(B.mb_info)[M.list_off + j];
  const int kind = info.x, cnt = info.z, head = info.w;
  const uint32_t key = (uint32_t)info.y;
  int rank = j;
  for (int q = 0; q < S.n_models; q++) {
    const int gq = S.model_off + q;
    if (gq == g) continue;
    const intf_model& Q = models[gq];
    rank += count_form_before(B.mb_t + Q.list_off, B.mb_info + 4ll * Q.list_off, B.n_mb[gq], t, kind, key);
  }
  const int ro = S.req_off;
  B.b_model[ro + rank] = mloc;
  B.b_size[ro + rank] = cnt;
  B.b_formed[ro + rank] = t;
  const int32_t* lrid = B.list_rid + M.list_off;
  for (int k = 0; k < cnt; k++) B.r_batch[ro + lrid[head + k]] = rank;
}
constexpr int kMergeWarps = 8;
__global__ void __launch_bounds__(32 * kMergeWarps) k_merge_batches_warp(const intf_scenario* __restrict__ scen,
                                                                         const intf_model* __restrict__ models,
                                                                         intf_replay_buffers B, int n_models) {
  const int g = blockIdx.x * kMergeWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (g >= n_models) return;
  const intf_model& M = models[g];
  const intf_scenario& S = scen[M.scen];
  const int n = B.n_mb[g];
  if (lane == 0 && n) atomicAdd(&B.n_batches[M.scen], n);
  for (int j = lane; j < n; j += 32) merge_batch(S, models, B, g, g - S.model_off, j);
}

// scenarios whose configuration the replay cannot run are flagged INTF_ST_CAP
__global__ void k_form_status(const intf_scenario* __restrict__ scen, int n_scen, intf_replay_buffers B) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_scen) return;
  const intf_scenario& S = scen[s];
  if (B.status[s] & INTF_ST_OVERFLOW) return;
  if (S.cap > B.cap_max || S.cap > kMaxCap || S.cap < 1 || S.max_bs < 1 || S.n_models > kMaxModels)
    B.status[s] |= INTF_ST_CAP;
}

// ---- K1b: noise draws of the first noise_k segments of every formed batch
// (`oracle.py:24-33`), fully parallel: takes the SeedSequence/PCG64/ziggurat/
// exp chain off the serial replay recurrence.  grid: (slots, scenarios).
// scenario owning packed request slot `slot` (req_off is increasing)
__device__ __forceinline__ int scen_of_slot(const intf_scenario* __restrict__ scen, int n_scen, long long slot) {
  int lo = 0, hi = n_scen - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (scen[mid].req_off <= slot) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Two launch shapes over the same draws: many scenarios -> one block per
// scenario (grid-stride over scenarios, looping over its formed batches x
// noise_k); few scenarios (long traces) -> grid-stride over the packed
// (request slot, draw) space, the owning scenario found by binary search.
constexpr int kPerScenarioMin = 4 * 148;  // below this many scenarios, flatten
__global__ void __launch_bounds__(256) k_noise_table(const intf_scenario* __restrict__ scen, int n_scen,
                                                     long long req_slots, intf_replay_buffers B) {
  const int K = B.noise_k;
  // concurrency_cap == 1: a batch runs alone as ONE segment, so the replay
  // (replay_cap1) reads only draw (b, 0): the other K - 1 are not computed
  if (n_scen >= kPerScenarioMin) {
    for (int s = blockIdx.x; s < n_scen; s += gridDim.x) {
      const intf_scenario& S = scen[s];
      const int Ks = S.cap == 1 ? 1 : K;
      double* out = B.noise_tab + (long long)S.req_off * K;
      // a thread per batch: its Ks draws share the SeedSequence work that does
      // not involve the segment index (noise_draws_k)
      for (long long b = threadIdx.x; b < B.n_batches[s]; b += blockDim.x)
        noise_draws_k(S.oracle_seed, S.batch_id_base + (uint64_t)b, Ks, S.sigma, out + b * K);
    }
    return;
  }
  for (long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x; slot < req_slots;
       slot += (long long)gridDim.x * blockDim.x) {
    const int s = scen_of_slot(scen, n_scen, slot);
    const intf_scenario& S = scen[s];
    const long long b = slot - S.req_off;
    if (b < B.n_batches[s])
      noise_draws_k(S.oracle_seed, S.batch_id_base + (uint64_t)b, S.cap == 1 ? 1 : K, S.sigma, B.noise_tab + slot * K);
  }
}

// ---- K2: the replay recurrence, one kReplayW-lane group per scenario (lane
// l < cap owns running slot l; replay_warp.cuh).
#ifndef INTF_REPLAY_WARPS
#define INTF_REPLAY_WARPS 4  // warps per k_replay_warp block
#endif
#ifndef INTF_JOB_WARPS
#define INTF_JOB_WARPS 1  // warps per busy-period job block (k_replay_jobs, k_jobs_replay)
#endif
// 12 resident replay warps per SM = 170 registers: no spills in the
// cap-templated replay (B200: C5 10^4 7.36 -> 6.77 ms at 3 blocks of 4 warps)
#ifndef INTF_REPLAY_MINB
#define INTF_REPLAY_MINB (12 / INTF_REPLAY_WARPS)
#endif
#define INTF_JOB_MINB (12 / INTF_JOB_WARPS)
constexpr int kReplayWarps = INTF_REPLAY_WARPS;
// Job kernels: a block keeps its registers until its LAST warp ends, so with
// one-warp blocks a long job does not hold finished warps' slots away from
// the next pass / trace (measured on C4: 3.04 -> 2.85 ms per trace, 2.00 ->
// 1.87 ms with two traces in flight; the C5 sweep kernel is better at 4,
// `profiles/replay_block_warps_r1k.txt`).
constexpr int kJobWarps = INTF_JOB_WARPS;
constexpr int kReplayW = 32;  // measured: one scenario per warp beats 4 x 8-lane groups (divergence)
// Replay order = longest-processing-time first by the device's own work
// estimate: formed batches, cap-1 scenarios weighted 1/5 (their max-plus chain
// is ~5x cheaper per batch).  A counting sort over 4,096 buckets (descending):
// histogram, one-block scan, scatter; `order` receives the permutation.
constexpr int kOrderBuckets = 4096;
__device__ __forceinline__ int order_bucket(const intf_scenario* scen, const intf_replay_buffers& B, int s) {
  const int nb = B.n_batches[s];
  const int w = scen[s].cap == 1 ? nb / 5 : nb;
  const int k = w / 2;
  return kOrderBuckets - 1 - (k < kOrderBuckets - 1 ? k : kOrderBuckets - 1);  // heavy -> bucket 0
}
__global__ void k_order_hist(const intf_scenario* __restrict__ scen, int n_scen, intf_replay_buffers B,
                             int32_t* __restrict__ cnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_scen) atomicAdd(&cnt[order_bucket(scen, B, s)], 1);
}
__global__ void __launch_bounds__(1024) k_order_scan(int32_t* __restrict__ cnt) {
  __shared__ int sh[1024];
  const int t = threadIdx.x;  // 4 buckets per thread
  int v[4], sum = 0;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    v[j] = cnt[4 * t + j];
    sum += v[j];
  }
  sh[t] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int x = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += x;
    __syncthreads();
  }
  int run = sh[t] - sum;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    cnt[4 * t + j] = run;
    run += v[j];
  }
}
__global__ void k_order_scatter(const intf_scenario* __restrict__ scen, int n_scen, intf_replay_buffers B,
                                int32_t* __restrict__ cnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_scen) B.order[atomicAdd(&cnt[order_bucket(scen, B, s)], 1)] = s;
}

// Persistent: one block per resident slot (INTF_REPLAY_MINB per SM); each warp
// pulls the next scenario index from a counter (B.slo_ws[0], free until the
// SLO pass) as soon as its previous scenario is done, so a long scenario
// never holds a block's other warps idle (block-granular scheduling would).
__global__ void __launch_bounds__(32 * kReplayWarps, INTF_REPLAY_MINB) k_replay_warp(const intf_scenario* __restrict__ scen,
                                                                    int n_scen, const intf_model* __restrict__ models,
                                                                    intf_table tab, intf_replay_buffers B) {
  __shared__ double sseg[kReplayWarps * (32 / kReplayW)][kMaxCap * kSmemSeg * 5];
  const int g = (threadIdx.x >> 5) * (32 / kReplayW) + ((threadIdx.x & 31) / kReplayW);
  for (;;) {
    int k = 0;
    if ((threadIdx.x & 31) == 0) k = atomicAdd(B.slo_ws, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= n_scen) return;
    const int s = B.order[k];  // longest-processing-time first (k_order_*)
    const int st0 = B.status[s];
    if (st0 & (INTF_ST_CAP | INTF_ST_OVERFLOW)) continue;
    const intf_scenario& S = scen[s];
    const ReplayJob J{s, 0, B.n_batches[s], S.seg_off, S.seg_cap, s};
    const ReplayJobOut r = replay_group<kReplayW>(J, scen, models, tab, B, sseg[g], st0);
    if ((threadIdx.x & (kReplayW - 1)) == 0) {
      B.n_segments[s] = r.n_segments;
      B.n_reseats[s] = r.n_reseats;
      B.status[s] = r.status;
    }
    __syncwarp();
  }
}

// ---- K2': busy-period segments of long traces.  Job i replays
// batches [lo[i], hi[i]) of scenario sc[i] from an idle GPU; its segment
// records go to S.seg_off + lo*(2cap-1) (a disjoint slice: a batch has at
// most 2cap-1 reseats), its outcome order to positions [lo, hi).
__global__ void __launch_bounds__(32 * kJobWarps, INTF_JOB_MINB) k_replay_jobs(const intf_scenario* __restrict__ scen,
                                                                    const intf_model* __restrict__ models,
                                                                    intf_table tab, intf_replay_buffers B,
                                                                    const int32_t* __restrict__ sc,
                                                                    const int32_t* __restrict__ lo,
                                                                    const int32_t* __restrict__ hi, int n_jobs,
                                                                    double* __restrict__ last_done,
                                                                    int32_t* __restrict__ info) {
  __shared__ double sseg[kJobWarps * (32 / kReplayW)][kMaxCap * kSmemSeg * 5];
  const int g = (threadIdx.x >> 5) * (32 / kReplayW) + ((threadIdx.x & 31) / kReplayW);
  const int i = blockIdx.x * kJobWarps * (32 / kReplayW) + g;
  if (i >= n_jobs) return;
  const int s = sc[i];
  const int st0 = B.status[s];
  const bool lead = (threadIdx.x & (kReplayW - 1)) == 0;
  if (st0 & (INTF_ST_CAP | INTF_ST_OVERFLOW)) {
    if (lead) info[3 * i] = st0;
    return;
  }
  const intf_scenario& S = scen[s];
  const int per = 2 * S.cap - 1;
  const ReplayJob J{s, lo[i], hi[i], S.seg_off + lo[i] * per, (hi[i] - lo[i]) * per, i};
  const ReplayJobOut r = replay_group<kReplayW>(J, scen, models, tab, B, sseg[g], 0);
  if (lead) {
    info[3 * i] = r.status;
    info[3 * i + 1] = r.n_segments;
    info[3 * i + 2] = r.n_reseats;
    last_done[i] = r.last_done;
  }
}

// ---- device-planned busy-period jobs (see intf_jobs in the header)
__global__ void __launch_bounds__(128) k_jobs_plan(const intf_scenario* __restrict__ scen, int n_scen,
                                                   const intf_model* __restrict__ models, intf_table tab,
                                                   intf_replay_buffers B, intf_jobs J) {
  const int s = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (s >= n_scen) return;
  const LaneGroup<32> G;
  const int lane = G.lane;
  const intf_scenario& S = scen[s];
  if (S.req_cap >= kBigJobs) return;  // k_jobs_plan_big
  const int nb = B.n_batches[s], ro = S.req_off, joff = J.joff[s], jcap = J.jcap[s];
  const intf_model* md = models + S.model_off;
  const bool bad = (B.status[s] & (INTF_ST_CAP | INTF_ST_OVERFLOW)) != 0;
  double carry = -INFINITY;  // max over earlier batches of formed + slow * solo
  int nj = 0;
  long long last_bucket = -1;
  if (!bad && nb > 0) {
    for (int base = 0; base < nb; base += 32) {
      const int b = base + lane;
      double f = 0.0, e = -INFINITY;
      if (b < nb) {
        f = B.b_formed[ro + b];
        const int entry = md[B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1;
        e = f + J.slow * tab.solo_ms[entry];
      }
      double incl = e;  // inclusive prefix max over the chunk (max is exact: order-free)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double v = G.shfl_up(incl, o);
        if (lane >= o) incl = incl > v ? incl : v;
      }
      double excl = G.shfl_up(incl, 1);
      if (lane == 0) excl = -INFINITY;
      const double before = carry > excl ? carry : excl;
      const bool cand = b < nb && (b == 0 || f > before);
      unsigned m = G.ballot(cand);
      while (m) {  // in batch order: one start per min_len bucket
        const int l = __ffs(m) - 1;
        m &= m - 1;
        const int bb = base + l;
        const long long bucket = bb / J.min_len;
        if (bb == 0 || bucket != last_bucket) {
          if (nj < jcap && lane == 0) J.lo[joff + nj] = bb;
          nj += nj < jcap ? 1 : 0;
          last_bucket = bucket;
        }
      }
      const double tot = G.shfl(incl, 31);
      carry = carry > tot ? carry : tot;
    }
  }
  if (lane == 0) {
    J.n_jobs[s] = nj;
    for (int j = 0; j < nj; j++) {
      J.hi[joff + j] = j + 1 < nj ? J.lo[joff + j + 1] : nb;
      J.dirty[joff + j] = 1;
      J.todo[atomicAdd(J.todo_count, 1)] = joff + j;
    }
    if (nj == 0) {  // nothing to replay: totals are zero
      B.n_segments[s] = 0;
      B.n_reseats[s] = 0;
    }
  }
}

// ---- long traces (req_cap >= kBigJobs): plan and verify with one 1024-thread
// block per scenario instead of one warp / one thread (a 10^6-request trace
// has ~4x10^5 batches and ~10^4 jobs).  Same decisions as k_jobs_plan /
// k_jobs_verify: the prefix maxima, first candidate per bucket, keep/merge
// pattern and compaction are computed with block scans.
constexpr int kBigThreads = 1024;

// block-wide exclusive scan (op = max for doubles, + for ints) of one value per thread
__device__ __forceinline__ double block_excl_max(double v, double* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int o = 1; o < kBigThreads; o <<= 1) {
    const double a = t >= o ? sh[t - o] : -INFINITY;
    __syncthreads();
    sh[t] = sh[t] > a ? sh[t] : a;
    __syncthreads();
  }
  const double r = t > 0 ? sh[t - 1] : -INFINITY;
  __syncthreads();
  return r;
}
__device__ __forceinline__ int block_excl_sum(int v, int* sh, int* total) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int o = 1; o < kBigThreads; o <<= 1) {
    const int a = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += a;
    __syncthreads();
  }
  const int r = t > 0 ? sh[t - 1] : 0;
  if (total) *total = sh[kBigThreads - 1];
  __syncthreads();
  return r;
}

// ---- K0a' (long lists), exact and parallel: the cumulative sum t += gap
// (`workload.py:91`) reproduced bit for bit without a 3x10^5-long add chain.
// Inside one binade [2^e, 2^(e+1)) every double is a multiple of u =
// 2^(e-52), so fl(t + g) = t + u * rint(g / u) as long as the sum stays in
// the binade and g / u is not a half-integer (ties-to-even would depend on
// t's last bit): a run of such steps is an exact INTEGER prefix sum.
//   k_bin_sums      (grid)  chunk c (32 gaps): S_c;
//   k_bin_scan      (block per model) T_c = sum of S before c: an estimate of
//                   t at the chunk start (a prediction only: all below is verified);
//   k_bin_classify  (grid)  chunk c is "clean" if [T_c - d, T_c + S_c + d]
//                   lies in one binade e (d bounds the estimate's error) and
//                   no gap is a half-integer multiple of u_e; N_c = sum rint(g / u_e);
//   k_bin_runs      (block per model) runs of clean chunks of one binade:
//                   segmented prefix sums P_c; one thread walks the runs and
//                   the other chunks in order: a run starting at the exact
//                   t_run ends at t_run + u P_last, verified inside [2^e,
//                   2^(e+1)) (so every intermediate sum was in the binade);
//                   anything else -- a binade crossing, a tie, a failed
//                   verification -- takes the 32 real fp64 adds per chunk;
//   k_bin_fill      (grid)  every run chunk's end t_run + u P_c (exact).
// Output: every 32nd partial sum in mb_t (ends), for k_fill_gaps.  mb_t is
// free until formation; per long model it holds (n32 = list_cap / 32 chunks)
// ends | S | T | P (int64) | code, evidx, evpos (int) | evT.
constexpr int kBinThreads = 1024;
constexpr int kBinOff = 2048;      // chunk code = e + kBinOff (clean), -1 (sequential)
constexpr int kBinHead = 1 << 20;  // code bit: first chunk of a run

struct BinScratch {
  double *ends, *S, *T, *evT;
  long long* P;
  int *code, *evidx, *evpos;
  int n32;
};
__device__ __forceinline__ BinScratch bin_scratch(const intf_model& M, const intf_replay_buffers& B) {
  BinScratch b;
  b.n32 = M.list_cap / kScanChunk;
  b.ends = B.mb_t + M.list_off;
  b.S = b.ends + b.n32;
  b.T = b.ends + 2 * b.n32;
  b.P = reinterpret_cast<long long*>(b.ends + 3 * b.n32);
  b.code = reinterpret_cast<int*>(b.ends + 4 * b.n32);
  b.evidx = b.code + b.n32;
  b.evpos = b.evidx + b.n32;
  b.evT = b.ends + 6 * b.n32;
  return b;
}

// grid (chunk blocks, models): a warp stages its 32 chunks (32 x 32 gaps)
// through shared memory with coalesced loads; lane l then owns chunk cb + l
constexpr int kBinWarps = 4;
__device__ __forceinline__ const intf_model* bin_model(const intf_model* models, int n_models_total) {
  const int g = blockIdx.z * gridDim.y + blockIdx.y;
  if (g >= n_models_total) return nullptr;
  const intf_model* M = models + g;
  return (M->list_cap < kBigList || M->rate_rps == 0.0) ? nullptr : M;
}
__device__ __forceinline__ int bin_stage(double (*sm)[33], const double* lt, int cb, int n32) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < 32; j++) {
    const int c = cb + j;
    sm[j][lane] = c < n32 ? lt[(long long)c * kScanChunk + lane] : 0.0;
  }
  __syncwarp();
  return cb + lane;
}

__global__ void __launch_bounds__(32 * kBinWarps) k_bin_sums(const intf_model* __restrict__ models, int n_models_total,
                                                             intf_replay_buffers B) {
  __shared__ double sm[kBinWarps][32][33];
  const intf_model* M = bin_model(models, n_models_total);
  if (!M) return;
  const BinScratch b = bin_scratch(*M, B);
  const int cb = (blockIdx.x * kBinWarps + (threadIdx.x >> 5)) * 32;
  if (cb >= b.n32) return;
  const int c = bin_stage(sm[threadIdx.x >> 5], B.list_t + M->list_off, cb, b.n32);
  double S = 0.0;
  for (int k = 0; k < kScanChunk; k++) S += sm[threadIdx.x >> 5][threadIdx.x & 31][k];
  if (c < b.n32) b.S[c] = S;
}

// block-wide inclusive scan (+) of one value per thread (1024 threads): warp
// shuffles, then the 32 warp totals; `tot` = the block total
template <typename V>
__device__ __forceinline__ V bin_block_incl(V v, V* sw, V* tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V a = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += a;
  }
  if (lane == 31) sw[w] = v;
  __syncthreads();
  if (w == 0) {
    V x = sw[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const V a = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += a;
    }
    sw[lane] = x;
  }
  __syncthreads();
  const V r = v + (w ? sw[w - 1] : V(0));
  *tot = sw[31];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kBinThreads) k_bin_scan(const intf_model* __restrict__ models, int n_models_total,
                                                          intf_replay_buffers B) {
  __shared__ double sw[32];
  const int g = blockIdx.x;
  if (g >= n_models_total) return;
  const intf_model& M = models[g];
  if (M.list_cap < kBigList || M.rate_rps == 0.0) return;
  const BinScratch b = bin_scratch(M, B);
  double carry = 0.0;
  for (int base = 0; base < b.n32; base += kBinThreads) {
    const int c = base + threadIdx.x;
    const double v = c < b.n32 ? b.S[c] : 0.0;
    double tot;
    const double incl = bin_block_incl(v, sw, &tot);
    if (c < b.n32) b.T[c] = carry + (incl - v);
    carry += tot;
  }
}

__global__ void __launch_bounds__(32 * kBinWarps) k_bin_classify(const intf_model* __restrict__ models,
                                                                 int n_models_total, intf_replay_buffers B) {
  __shared__ double sm[kBinWarps][32][33];
  const intf_model* M = bin_model(models, n_models_total);
  if (!M) return;
  const BinScratch b = bin_scratch(*M, B);
  const int cb = (blockIdx.x * kBinWarps + (threadIdx.x >> 5)) * 32;
  if (cb >= b.n32) return;
  const int c = bin_stage(sm[threadIdx.x >> 5], B.list_t + M->list_off, cb, b.n32);
  if (c >= b.n32) return;
  const double T = b.T[c], hi_est = T + b.S[c];
  const double d = hi_est * 0x1p-40 + 4.0 * M->list_cap * ldexp(1.0, ilogb(hi_est > 0.0 ? hi_est : 1.0) - 52);
  int cd = -1;
  long long N = 0;
  if (c > 0 && T - d > 0.0 && ilogb(T - d) == ilogb(hi_est + d)) {
    const int e = ilogb(T - d);
    const double inv = ldexp(1.0, 52 - e);
    bool ok = true;
    for (int k = 0; k < kScanChunk; k++) {
      const double x = sm[threadIdx.x >> 5][threadIdx.x & 31][k] * inv;
      const double r = rint(x);
      ok &= x < 0x1p53 && fabs(x - r) != 0.5;
      N += (long long)r;
    }
    if (ok) cd = e + kBinOff;
  }
  b.code[c] = cd;
  b.P[c] = N;
}

__global__ void __launch_bounds__(kBinThreads) k_bin_runs(const intf_model* __restrict__ models, int n_models_total,
                                                          intf_replay_buffers B) {
  __shared__ long long swl[32];
  __shared__ int swf[32], swi[32];
  __shared__ long long shl[kBinThreads];
  __shared__ int shf[kBinThreads], shc[kBinThreads], shn[kBinThreads];
  const int g = blockIdx.x;
  if (g >= n_models_total) return;
  const intf_model& M = models[g];
  if (M.list_cap < kBigList || M.rate_rps == 0.0) return;
  const BinScratch b = bin_scratch(M, B);
  const int n32 = b.n32, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const double* lt = B.list_t + M.list_off;
  // runs: head = clean and (first chunk, or the previous chunk is not of
  // this run); segmented inclusive prefix sums of N (P, in place); events
  // (sequential chunks and run heads) compacted in order
  long long run = 0;  // the open run's sum carried across rounds
  int evbase = 0;
  for (int base = 0; base < n32; base += kBinThreads) {
    const int c = base + t;
    int cd = -1, head = 1;
    long long v = 0;
    if (c < n32) {
      cd = b.code[c];
      v = b.P[c];
      head = cd < 0 || c == 0 || (b.code[c - 1] & ~kBinHead) != cd;  // (the previous round may have set its head bit)
    }
    // warp segmented scan
    int f = head;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long a = __shfl_up_sync(0xffffffffu, v, o);
      const int af = __shfl_up_sync(0xffffffffu, f, o);
      if (lane >= o) {
        if (!f) v += a;
        f |= af;
      }
    }
    if (lane == 31) {
      swl[w] = v;
      swf[w] = f;
    }
    __syncthreads();
    if (w == 0) {  // exclusive segmented scan of the warp aggregates, seeded by the carried run
      long long x = swl[lane];
      int xf = swf[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long a = __shfl_up_sync(0xffffffffu, x, o);
        const int af = __shfl_up_sync(0xffffffffu, xf, o);
        if (lane >= o) {
          if (!xf) x += a;
          xf |= af;
        }
      }
      // exclusive: the aggregate before warp `lane`, incl. the carry
      long long ex = __shfl_up_sync(0xffffffffu, x, 1);
      int exf = __shfl_up_sync(0xffffffffu, xf, 1);
      if (lane == 0) ex = 0, exf = 0;
      swl[lane] = exf ? ex : run + ex;
      swf[lane] = xf;  // inclusive flag of warps 0..lane (for the next carry)
    }
    __syncthreads();
    const long long incl = f ? v : swl[w] + v;
    // events
    const int fe = c < n32 && (cd < 0 || head);
    int etot;
    const int eincl = bin_block_incl(fe, swi, &etot);
    if (c < n32) {
      b.P[c] = incl;
      b.evidx[c] = evbase + eincl - 1;
      if (fe) b.evpos[evbase + eincl - 1] = c;
    }
    // the next round's carry: the last chunk's inclusive value
    if (t == kBinThreads - 1) shl[0] = incl;
    __syncthreads();
    run = shl[0];
    evbase += etot;
    __syncthreads();
    if (c < n32 && cd >= 0 && head) b.code[c] = cd | kBinHead;
  }
  __syncthreads();
  // the walk over events (one thread; each batch of events staged in shared
  // memory first)
  double tc = 0.0;
  for (int b0 = 0; b0 < evbase; b0 += kBinThreads) {
    const int i = b0 + t;
    if (i < evbase) {
      const int c = b.evpos[i], nxt = i + 1 < evbase ? b.evpos[i + 1] : n32;
      shc[t] = c;
      shn[t] = nxt;
      shf[t] = b.code[c];
      shl[t] = b.P[nxt - 1];
    }
    __syncthreads();
    if (t == 0) {
      const int nb = min(kBinThreads, evbase - b0);
      for (int k = 0; k < nb; k++) {
        const int cd = shf[k];
        bool walked = true;
        if (cd >= 0) {
          const int e = (cd & ~kBinHead) - kBinOff;
          const double te = tc + ldexp(1.0, e - 52) * (double)shl[k];
          if (tc >= ldexp(1.0, e) && te < ldexp(1.0, e + 1)) {
            b.evT[b0 + k] = tc;
            tc = te;
            walked = false;
          }
        }
        if (walked) {
          b.evT[b0 + k] = NAN;
          for (int cc = shc[k]; cc < shn[k]; cc++) {
            double gv[kScanChunk];
#pragma unroll
            for (int q = 0; q < kScanChunk; q++) gv[q] = lt[cc * kScanChunk + q];
#pragma unroll
            for (int q = 0; q < kScanChunk; q++) tc = tc + gv[q];
            b.ends[cc] = tc;
          }
        }
      }
    }
    __syncthreads();
  }
}

__global__ void k_bin_fill(const intf_model* __restrict__ models, int n_models_total, intf_replay_buffers B) {
  const intf_model* M = bin_model(models, n_models_total);
  if (!M) return;
  const BinScratch b = bin_scratch(*M, B);
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= b.n32) return;
  const int i = b.evidx[c];
  const double trun = b.evT[i];
  if (isnan(trun)) return;  // walked: already exact
  const int e = (b.code[b.evpos[i]] & ~kBinHead) - kBinOff;
  b.ends[c] = trun + ldexp(1.0, e - 52) * (double)b.P[c];
}

__global__ void __launch_bounds__(kBigThreads) k_jobs_plan_big(const intf_scenario* __restrict__ scen,
                                                               const intf_model* __restrict__ models, intf_table tab,
                                                               intf_replay_buffers B, intf_jobs J) {
  __shared__ double shd[kBigThreads];
  __shared__ int shi[kBigThreads];
  __shared__ int todo_base;
  const int s = blockIdx.x;
  const intf_scenario& S = scen[s];
  if (S.req_cap < kBigJobs) return;
  const int t = threadIdx.x;
  const int nb = B.n_batches[s], ro = S.req_off, joff = J.joff[s], jcap = J.jcap[s];
  const bool bad = (B.status[s] & (INTF_ST_CAP | INTF_ST_OVERFLOW)) != 0;
  const intf_model* md = models + S.model_off;
  const int n = bad ? 0 : nb;
  const int R = (n + kBigThreads - 1) / kBigThreads, b0 = t * R, b1 = min(n, b0 + R);
  const int nbk = (n + J.min_len - 1) / J.min_len;
  int* first = reinterpret_cast<int*>(J.scratch + 6ll * joff);  // [nbk <= 12 jcap] first candidate per bucket
  for (int k = t; k < nbk; k += kBigThreads) first[k] = 0x7fffffff;
  // pass 1: max of formed + slow*solo over this thread's range
  double m = -INFINITY;
  for (int b = b0; b < b1; b++) {
    const double e = B.b_formed[ro + b] + J.slow * tab.solo_ms[md[B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1];
    m = m > e ? m : e;
  }
  double before = block_excl_max(m, shd);  // also orders the first[] initialisation before the atomics
  // pass 2: candidates (forming after every earlier batch's optimistic end)
  for (int b = b0; b < b1; b++) {
    const double f = B.b_formed[ro + b];
    const double e = f + J.slow * tab.solo_ms[md[B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1];
    if (b == 0 || f > before) atomicMin(&first[b / J.min_len], b);
    before = before > e ? before : e;
  }
  __syncthreads();
  // pass 3: the first candidate of every bucket starts a job (compaction)
  const int K = (nbk + kBigThreads - 1) / kBigThreads, k0 = t * K, k1 = min(nbk, k0 + K);
  int cnt = 0;
  for (int k = k0; k < k1; k++) cnt += first[k] != 0x7fffffff;
  int total = 0;
  int r = block_excl_sum(cnt, shi, &total);
  for (int k = k0; k < k1; k++)
    if (first[k] != 0x7fffffff) {
      if (r < jcap) J.lo[joff + r] = first[k];
      r++;
    }
  const int nj = total < jcap ? total : jcap;
  if (t == 0) {
    J.n_jobs[s] = nj;
    todo_base = nj ? atomicAdd(J.todo_count, nj) : 0;
    if (nj == 0) {
      B.n_segments[s] = 0;
      B.n_reseats[s] = 0;
    }
  }
  __syncthreads();
  for (int j = t; j < nj; j += kBigThreads) {
    J.hi[joff + j] = j + 1 < nj ? J.lo[joff + j + 1] : nb;
    J.dirty[joff + j] = 1;
    J.todo[todo_base + j] = joff + j;
  }
}

// ---- the same plan, grid-parallel (C4's ~4x10^5 batches over ~200 blocks):
// p1 block maxima of formed + slow*solo, p2 exclusive scan of the maxima,
// p3 candidates -> first candidate per bucket, p4 compaction (one block).
constexpr int kPlanChunk = 2048;  // batches per block (256 threads x 8)
__device__ __forceinline__ double plan_e(const intf_scenario& S, const intf_model* md, const intf_table& tab,
                                         const intf_replay_buffers& B, double slow, int b) {
  const int ro = S.req_off;
  return B.b_formed[ro + b] + slow * tab.solo_ms[md[B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1];
}
__global__ void __launch_bounds__(256) k_plan_p1(const intf_scenario* __restrict__ scen,
                                                 const intf_model* __restrict__ models, intf_table tab,
                                                 intf_replay_buffers B, intf_jobs J) {
  __shared__ double red[256];
  const int s = blockIdx.y;
  const intf_scenario& S = scen[s];
  if (S.req_cap < kBigJobs) return;
  const int nb = (B.status[s] & (INTF_ST_CAP | INTF_ST_OVERFLOW)) ? 0 : B.n_batches[s];
  const int b0 = blockIdx.x * kPlanChunk;
  if (b0 >= max(nb, 1)) return;
  const int joff = J.joff[s], jcap = J.jcap[s];
  int* first = reinterpret_cast<int*>(J.scratch + 6ll * joff);
  double* bmax = J.scratch + 6ll * joff + jcap;
  const int k0 = b0 / J.min_len, k1 = min((b0 + kPlanChunk - 1) / J.min_len, (nb - 1) / J.min_len);
  for (int k = k0 + threadIdx.x; k <= k1; k += blockDim.x) first[k] = 0x7fffffff;
  const intf_model* md = models + S.model_off;
  double m = -INFINITY;
  for (int i = 0; i < kPlanChunk / 256; i++) {
    const int b = b0 + threadIdx.x * (kPlanChunk / 256) + i;
    if (b < nb) {
      const double e = plan_e(S, md, tab, B, J.slow, b);
      m = m > e ? m : e;
    }
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = red[threadIdx.x] > red[threadIdx.x + o] ? red[threadIdx.x] : red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) bmax[blockIdx.x] = red[0];
}
__global__ void __launch_bounds__(kBigThreads) k_plan_p2(const intf_scenario* __restrict__ scen,
                                                         intf_replay_buffers B, intf_jobs J) {
  __shared__ double shd[kBigThreads];
  const int s = blockIdx.x;
  if (scen[s].req_cap < kBigJobs) return;
  const int nb = (B.status[s] & (INTF_ST_CAP | INTF_ST_OVERFLOW)) ? 0 : B.n_batches[s];
  const int nblk = (nb + kPlanChunk - 1) / kPlanChunk;
  double* bmax = J.scratch + 6ll * J.joff[s] + J.jcap[s];
  // exclusive max-scan in place, kBigThreads entries per round
  double carry = -INFINITY;
  for (int base = 0; base < nblk; base += kBigThreads) {
    const int i = base + threadIdx.x;
    const double v = i < nblk ? bmax[i] : -INFINITY;
    const double ex = block_excl_max(v, shd);
    const double pre = carry > ex ? carry : ex;
    if (i < nblk) bmax[i] = pre;
    const double incl = pre > v ? pre : v;
    shd[threadIdx.x] = incl;
    __syncthreads();
    carry = shd[kBigThreads - 1];
    __syncthreads();
  }
}
__global__ void __launch_bounds__(256) k_plan_p3(const intf_scenario* __restrict__ scen,
                                                 const intf_model* __restrict__ models, intf_table tab,
                                                 intf_replay_buffers B, intf_jobs J) {
  __shared__ double sh[256];
  const int s = blockIdx.y;
  const intf_scenario& S = scen[s];
  if (S.req_cap < kBigJobs) return;
  const int nb = (B.status[s] & (INTF_ST_CAP | INTF_ST_OVERFLOW)) ? 0 : B.n_batches[s];
  const int b0 = blockIdx.x * kPlanChunk;
  if (b0 >= nb) return;
  const int joff = J.joff[s], jcap = J.jcap[s];
  int* first = reinterpret_cast<int*>(J.scratch + 6ll * joff);
  const double* bmax = J.scratch + 6ll * joff + jcap;
  const intf_model* md = models + S.model_off;
  constexpr int PER = kPlanChunk / 256;
  const int bt = b0 + threadIdx.x * PER;
  double e[PER], m = -INFINITY;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    e[i] = bt + i < nb ? plan_e(S, md, tab, B, J.slow, bt + i) : -INFINITY;
    m = m > e[i] ? m : e[i];
  }
  // exclusive max over earlier threads of the block (Hillis-Steele), then the block's prefix
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const double a = threadIdx.x >= o ? sh[threadIdx.x - o] : -INFINITY;
    __syncthreads();
    sh[threadIdx.x] = sh[threadIdx.x] > a ? sh[threadIdx.x] : a;
    __syncthreads();
  }
  double before = threadIdx.x ? sh[threadIdx.x - 1] : -INFINITY;
  before = before > bmax[blockIdx.x] ? before : bmax[blockIdx.x];
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int b = bt + i;
    if (b >= nb) break;
    if (b == 0 || B.b_formed[S.req_off + b] > before) atomicMin(&first[b / J.min_len], b);
    before = before > e[i] ? before : e[i];
  }
}
__global__ void __launch_bounds__(kBigThreads) k_plan_p4(const intf_scenario* __restrict__ scen, intf_replay_buffers B,
                                                         intf_jobs J) {
  __shared__ int shi[kBigThreads];
  __shared__ int todo_base;
  const int s = blockIdx.x;
  const intf_scenario& S = scen[s];
  if (S.req_cap < kBigJobs) return;
  const int t = threadIdx.x;
  const int nb = (B.status[s] & (INTF_ST_CAP | INTF_ST_OVERFLOW)) ? 0 : B.n_batches[s];
  const int joff = J.joff[s], jcap = J.jcap[s];
  const int* first = reinterpret_cast<const int*>(J.scratch + 6ll * joff);
  const int nbk = (nb + J.min_len - 1) / J.min_len;
  const int K = (nbk + kBigThreads - 1) / kBigThreads, k0 = t * K, k1 = min(nbk, k0 + K);
  int cnt = 0;
  for (int k = k0; k < k1; k++) cnt += first[k] != 0x7fffffff;
  int total = 0;
  int r = block_excl_sum(cnt, shi, &total);
  for (int k = k0; k < k1; k++)
    if (first[k] != 0x7fffffff) {
      if (r < jcap) J.lo[joff + r] = first[k];
      r++;
    }
  const int nj = total < jcap ? total : jcap;
  if (t == 0) {
    J.n_jobs[s] = nj;
    todo_base = nj ? atomicAdd(J.todo_count, nj) : 0;
    if (nj == 0) {
      B.n_segments[s] = 0;
      B.n_reseats[s] = 0;
    }
  }
  __syncthreads();
  for (int j = t; j < nj; j += kBigThreads) {
    J.hi[joff + j] = j + 1 < nj ? J.lo[joff + j + 1] : nb;
    J.dirty[joff + j] = 1;
    J.todo[todo_base + j] = joff + j;
  }
}

// Verify of a long trace (`replay_segmented_host`'s check, block-parallel):
// boundary j fails iff the previous job (each job's last completion from its
// own start) ends after job j's first formation; failing jobs join the kept
// job before them (whole runs at once), and a holding boundary behind a
// merged job is checked again next pass.  Tiles of kVerR rows x kVerThreads
// jobs (job = base + row * kVerThreads + thread: coalesced loads and
// stores), every field of a thread's jobs held in registers (all loads
// issued together), the kept jobs ranked by warp ballots + one warp scan of
// the per-(row, warp) counts, and compacted IN PLACE: a kept job's rank never
// exceeds its index, so a tile only overwrites slots below its own first job
// (the slot just below holds either that same job or a later tile's, not yet
// written), and every read of the tile precedes the barrier before its writes.
constexpr int kVerThreads = 512, kVerR = 12, kVerWarps = kVerThreads / 32;
constexpr int kVerWords = kVerR * kVerWarps;  // one ballot word per (row, warp)
static_assert(kVerWords <= 32 * 8, "k_jobs_verify_big: one warp scans the (row, warp) counts, <= 8 per lane");
__global__ void __launch_bounds__(kVerThreads) k_jobs_verify_big(const intf_scenario* __restrict__ scen,
                                                                 intf_replay_buffers B, intf_jobs J) {
  __shared__ unsigned fwd[kVerWords];  // failing boundaries, bit = tile position & 31
  __shared__ int koff[kVerWords];      // kept jobs before each (row, warp) word in the tile
  __shared__ int tile_kept, next_fails, any_fail, tot_segs, tot_res, last_hi;
  const int s = blockIdx.x;
  const intf_scenario& S = scen[s];
  if (S.req_cap < kBigJobs) return;
  const int n = J.n_jobs[s], joff = J.joff[s];
  if (n == 0) return;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, ro = S.req_off;
  const unsigned lt = (1u << lane) - 1u;
  if (t == 0) {
    last_hi = J.hi[joff + n - 1];
    tot_segs = tot_res = any_fail = 0;
  }
  auto fails = [&](int j, int l, int h, double pv) -> bool {
    return j > 0 && !(h <= l || pv <= B.b_formed[ro + l]);
  };
  int w = 0;  // kept jobs so far (block-uniform)
  int st = 0, segs = 0, res = 0;
  for (int base = 0; base < n; base += kVerThreads * kVerR) {
    const int tn = min(n - base, kVerThreads * kVerR);
    int lo[kVerR], i0[kVerR], i1[kVerR], i2[kVerR];
    double last[kVerR];
    unsigned fm = 0u, vm = 0u;  // bit k: row k's job fails / exists
#pragma unroll
    for (int k = 0; k < kVerR; k++) {
      const int p = k * kVerThreads + t, sj = joff + base + p;
      if (p < tn) {
        lo[k] = J.lo[sj];
        const int h = J.hi[sj];
        const double pv = base + p > 0 ? J.last[sj - 1] : -INFINITY;
        last[k] = J.last[sj];
        i0[k] = J.info[3 * sj];
        i1[k] = J.info[3 * sj + 1];
        i2[k] = J.info[3 * sj + 2];
        vm |= 1u << k;
        if (fails(base + p, lo[k], h, pv)) fm |= 1u << k;
      }
    }
    if (t == 0) {  // the next tile's first boundary (the absorb flag of this tile's last job)
      const int j = base + tn, sj = joff + j;
      next_fails = j < n && fails(j, J.lo[sj], J.hi[sj], J.last[sj - 1]);
    }
#pragma unroll
    for (int k = 0; k < kVerR; k++) {
      const unsigned bf = __ballot_sync(0xffffffffu, (fm >> k) & 1u);
      const unsigned bk = __ballot_sync(0xffffffffu, ((vm & ~fm) >> k) & 1u);
      if (lane == 0) {
        fwd[k * kVerWarps + wid] = bf;
        koff[k * kVerWarps + wid] = __popc(bk);
      }
    }
    __syncthreads();  // (every read of the tile done)
    if (wid == 0) {  // exclusive scan of the per-word kept counts, in job order
      constexpr int per = (kVerWords + 31) / 32;
      int c[per], sum = 0;
      unsigned f = 0u;
#pragma unroll
      for (int i = 0; i < per; i++) {
        const int q = lane * per + i;
        c[i] = q < kVerWords ? koff[q] : 0;
        f |= q < kVerWords ? fwd[q] : 0u;
        sum += c[i];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int run = incl - sum;
#pragma unroll
      for (int i = 0; i < per; i++) {
        const int q = lane * per + i;
        if (q < kVerWords) koff[q] = run;
        run += c[i];
      }
      if (lane == 31) tile_kept = incl;
      if (__any_sync(0xffffffffu, f != 0u) && lane == 0) any_fail = 1;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kVerR; k++) {
      const int p = k * kVerThreads + t, word = k * kVerWarps + wid;
      const bool kept = ((vm & ~fm) >> k) & 1u;
      const unsigned bk = __ballot_sync(0xffffffffu, kept);
      // the boundary after job p: the next lane, the next word's bit 0, or the next tile
      const bool absorbs = p + 1 < tn ? ((fwd[(p + 1) >> 5] >> ((p + 1) & 31)) & 1u) != 0u : next_fails != 0;
      const bool dirty = kept && absorbs;
      const int r = w + koff[word] + __popc(bk & lt);
      if (kept) {
        const int dj = joff + r;
        J.lo[dj] = lo[k];
        J.last[dj] = last[k];
        J.info[3 * dj] = i0[k];
        J.info[3 * dj + 1] = i1[k];
        J.info[3 * dj + 2] = i2[k];
        J.dirty[dj] = dirty ? 1 : 0;
        st |= i0[k];
        segs += i1[k];
        res += dirty ? 0 : i2[k];
      }
      // a dirty job exists iff some boundary failed: queue it now (replay order is immaterial)
      const unsigned bd = __ballot_sync(0xffffffffu, dirty);
      if (bd) {
        int at = 0;
        if (lane == 0) at = atomicAdd(J.todo_count, __popc(bd));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (dirty) J.todo[at + __popc(bd & lt)] = joff + r;
      }
    }
    w += tile_kept;
    __syncthreads();  // the tile's writes land before the next tile reads the slot below it
  }
  // hi of each kept job = lo of the next kept job
  for (int q = t; q < w; q += kVerThreads) J.hi[joff + q] = q + 1 < w ? J.lo[joff + q + 1] : last_hi;
  if (t == 0) J.n_jobs[s] = w;
  if (any_fail) return;  // merged jobs queued: totals after the next pass
  // every boundary holds: per-scenario totals
  const int st_w = (int)__reduce_or_sync(0xffffffffu, (unsigned)st);
  const int segs_w = __reduce_add_sync(0xffffffffu, segs), res_w = __reduce_add_sync(0xffffffffu, res);
  if (lane == 0) {
    if (st_w) atomicOr(&B.status[s], st_w);
    atomicAdd(&tot_segs, segs_w);
    atomicAdd(&tot_res, res_w);
  }
  __syncthreads();
  if (t == 0) {
    B.n_segments[s] = tot_segs;
    B.n_reseats[s] = tot_res;
  }
}

__global__ void __launch_bounds__(32 * kJobWarps, INTF_JOB_MINB) k_jobs_replay(const intf_scenario* __restrict__ scen,
                                                                    const intf_model* __restrict__ models,
                                                                    intf_table tab, intf_replay_buffers B,
                                                                    intf_jobs J, int n_todo) {
  __shared__ double sseg[kJobWarps * (32 / kReplayW)][kMaxCap * kSmemSeg * 5];
  const int g = (threadIdx.x >> 5) * (32 / kReplayW) + ((threadIdx.x & 31) / kReplayW);
  // n_todo < 0: the count is the device's (*J.todo_count, set by the plan /
  // the last verify), so passes can be queued without a host round trip
  const int n = n_todo >= 0 ? n_todo : *J.todo_count;
  const int stride = gridDim.x * kJobWarps * (32 / kReplayW);
  // host count: a warp per entry (the hardware schedules the blocks as warps
  // free up); device count (a one-wave grid): each warp takes the next entry
  // from todo_count[1] when its job is done, so the longest-first list stays
  // balanced
  auto next = [&](int cur) -> int {
    if (n_todo >= 0) return cur + stride;
    int k = 0;
    if ((threadIdx.x & 31) == 0) k = atomicAdd(J.todo_count + 1, 1);
    return __shfl_sync(0xffffffffu, k, 0);
  };
  for (int k = n_todo >= 0 ? blockIdx.x * kJobWarps * (32 / kReplayW) + g : next(0); k < n; k = next(k)) {
    const int slot = J.todo[k];
    const int s = J.slot_scen[slot];
    const intf_scenario& S = scen[s];
    const int per = 2 * S.cap - 1;
    const int jlo = J.lo[slot], jhi = J.hi[slot];
    if (jlo < J.own_lo || jlo >= J.own_hi) {  // another rank's job: neutral for the MAX all_reduce
      if ((threadIdx.x & (kReplayW - 1)) == 0) {
        J.info[3 * slot] = J.info[3 * slot + 1] = J.info[3 * slot + 2] = 0;
        J.last[slot] = -INFINITY;
        J.dirty[slot] = 0;
      }
      continue;
    }
    const ReplayJob RJ{s, jlo, jhi, S.seg_off + jlo * per, (jhi - jlo) * per, k};
    const ReplayJobOut r = replay_group<kReplayW>(RJ, scen, models, tab, B, sseg[g], 0);
    if ((threadIdx.x & (kReplayW - 1)) == 0) {
      J.info[3 * slot] = r.status;
      J.info[3 * slot + 1] = r.n_segments;
      J.info[3 * slot + 2] = r.n_reseats;
      J.last[slot] = r.last_done;
      J.dirty[slot] = 0;
    }
  }
}

// one thread per scenario: check boundaries in order, merge failing jobs into
// their predecessor (compacting the scenario's slots), queue merged jobs
__global__ void k_jobs_verify(const intf_scenario* __restrict__ scen, int n_scen, intf_replay_buffers B,
                              intf_jobs J) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_scen) return;
  const intf_scenario& S = scen[s];
  if (S.req_cap >= kBigJobs) return;  // k_jobs_verify_big
  const int n = J.n_jobs[s], joff = J.joff[s], ro = S.req_off;
  if (n == 0) return;
  int w = 0;  // write cursor (kept jobs)
  bool failed = false;
  for (int j = 0; j < n; j++) {
    const int sj = joff + j;
    bool keep = true;
    if (j > 0) {
      // job j-1's own last completion (from its own start; slot sj-1 is not
      // yet overwritten by the compaction).  A failing boundary merges job j
      // into the kept job before it -- whole runs of failures at once; a
      // holding boundary behind a merged job is checked again next pass
      // against the merged job's fresh last completion.
      const double prev_last = J.last[sj - 1];
      keep = J.hi[sj] <= J.lo[sj] || prev_last <= B.b_formed[ro + J.lo[sj]];
    }
    if (keep) {
      const int dw = joff + w;
      if (dw != sj) {
        J.lo[dw] = J.lo[sj];
        J.hi[dw] = J.hi[sj];
        J.last[dw] = J.last[sj];
        J.info[3 * dw] = J.info[3 * sj];
        J.info[3 * dw + 1] = J.info[3 * sj + 1];
        J.info[3 * dw + 2] = J.info[3 * sj + 2];
        J.dirty[dw] = 0;
      }
      w++;
    } else {  // boundary j fails: job j joins the previous kept job
      const int dp = joff + w - 1;
      J.hi[dp] = J.hi[sj];
      J.dirty[dp] = 1;
      failed = true;
    }
  }
  J.n_jobs[s] = w;
  if (failed) {
    for (int j = 0; j < w; j++)
      if (J.dirty[joff + j]) J.todo[atomicAdd(J.todo_count, 1)] = joff + j;
    return;
  }
  int st = B.status[s], segs = 0, res = 0;
  for (int j = 0; j < w; j++) {
    st |= J.info[3 * (joff + j)];
    segs += J.info[3 * (joff + j) + 1];
    res += J.info[3 * (joff + j) + 2];
  }
  B.status[s] = st;
  B.n_segments[s] = segs;
  B.n_reseats[s] = res;
}

// ---- K3: SLO records + per-model nearest-rank percentiles, one block per
// scenario.  Percentiles by MSB radix select on v = key - base, the latency
// bits (latency >= 0, so IEEE bit order == numeric order) offset by the
// scenario's smallest key: base = (min of the keys' high words) << 32 and
// v < 2^T with T = 32 + bit length of the high words' span, so the first
// 8-bit digit (bits T-1..T-8) spreads over the range actually used (starting
// at bit 63, one pass would hold every record in one bin: latencies on both
// sides of 2 ms already differ in bit 62).  The first pass's histogram is
// shared by the three quantiles (same empty prefix); in the cached path the
// records still matching a quantile's prefix are compacted after each pass,
// and once every (model, quantile)'s selected bin holds <= kSloFinish records
// one warp per (model, quantile) ranks them directly.
#ifndef INTF_SLO_THREADS
#define INTF_SLO_THREADS 256
#endif
constexpr int kSloThreads = INTF_SLO_THREADS;
constexpr int kSloGroup = 4;          // models per radix pass group (smem: 12 KB of histograms)
constexpr int kSloBigReq = 1 << 16;  // above this request capacity: grid-wide SLO passes
#ifndef INTF_SLO_CACHE
#define INTF_SLO_CACHE 2048
#endif
constexpr int kSloCache = INTF_SLO_CACHE;  // records whose latency keys k_slo keeps in shared memory (26 KB with indices)
constexpr int kSloFinish = 32;       // a selected bin this small is ranked by one warp
#ifndef INTF_SLO_UNROLL
#define INTF_SLO_UNROLL 4
#endif
constexpr int kSloUnroll = INTF_SLO_UNROLL;  // records per thread whose loads are issued together

__device__ __forceinline__ unsigned long long lat_key(double v) {
  unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_lat(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
// digit of v at [shift, shift + 8) (shift < 0: the low bits, left-aligned)
__device__ __forceinline__ unsigned slo_digit(unsigned long long v, int shift) {
  return (unsigned)((shift >= 0 ? v >> shift : v << -shift) & 0xffull);
}
__device__ __forceinline__ unsigned long long slo_put(unsigned d, int shift) {
  return shift >= 0 ? (unsigned long long)d << shift : (unsigned long long)(d >> -shift);
}
// v agrees with prefix pv on every bit at or above `from` (from >= 64: no bits)
__device__ __forceinline__ bool slo_match(unsigned long long v, unsigned long long pv, int from) {
  return from >= 64 || ((v ^ pv) >> (from > 0 ? from : 0)) == 0ull;
}

__global__ void __launch_bounds__(kSloThreads) k_slo(const intf_scenario* __restrict__ scen,
                                                     const intf_model* __restrict__ models, intf_replay_buffers B,
                                                     const double* __restrict__ warm_cutoff, int32_t* out_n,
                                                     int32_t* out_met, double* out_p) {
  const int s = blockIdx.x;
  const intf_scenario S = scen[s];
  const int n = B.n_req[s];
  const int ro = S.req_off;
  __shared__ int cnt_n[kMaxModels], cnt_met[kMaxModels];
  __shared__ unsigned int hist[kSloGroup][3][256];
  __shared__ unsigned long long prefix[kSloGroup][3];
  __shared__ int rank_left[kSloGroup][3];
  __shared__ int use_all;
  __shared__ unsigned hi_min, hi_max;
  __shared__ unsigned long long fin[kSloThreads / 32][kSloFinish];
  if ((B.status[s] & (INTF_ST_OVERFLOW | INTF_ST_SEG_STRIDE)) || S.n_models > kMaxModels) return;
  const double cutoff = warm_cutoff ? warm_cutoff[s] : -INFINITY;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = threadIdx.x; m < kMaxModels; m += blockDim.x) cnt_n[m] = cnt_met[m] = 0;
  if (threadIdx.x == 0) {
    use_all = 0;
    hi_min = 0xffffffffu;
    hi_max = 0u;
  }
  __syncthreads();
  // latency keys (and model ids) of the trimmed records, cached in shared
  // memory when they fit (kSloCache records): the radix passes re-read shared
  // memory, not four global arrays.  Cached path: the records still matching
  // one of the group's quantile prefixes, compacted after every radix pass
  // (double-buffered index lists), so later passes touch a few percent.
  extern __shared__ unsigned long long kcache[];
  unsigned char* mcache = reinterpret_cast<unsigned char*>(kcache + kSloCache);
  unsigned short* cand[2] = {reinterpret_cast<unsigned short*>(mcache + kSloCache),
                             reinterpret_cast<unsigned short*>(mcache + kSloCache) + kSloCache};
  __shared__ int n_cand[2];
  __shared__ int unresolved[2];  // by pass parity: pass p's check and pass p+1's reset never share a word
  const bool cached = n <= kSloCache;
  // one pass over the records (`simcore.py:264-279`): SLO flags, counts, key
  // cache, key range; kSloUnroll records per thread with their loads together
  unsigned kmin = 0xffffffffu, kmax = 0u;
  for (int i0 = 0; i0 < n; i0 += kSloUnroll * kSloThreads) {
    int bb[kSloUnroll], mm[kSloUnroll];
    double at[kSloUnroll], bc[kSloUnroll];
#pragma unroll
    for (int u = 0; u < kSloUnroll; u++) {
      const int i = i0 + u * kSloThreads + threadIdx.x;
      if (i < n) {
        bb[u] = B.r_batch[ro + i];
        at[u] = B.arr_t[ro + i];
        mm[u] = B.arr_model[ro + i];
      }
    }
#pragma unroll
    for (int u = 0; u < kSloUnroll; u++) {
      const int i = i0 + u * kSloThreads + threadIdx.x;
      if (i < n) bc[u] = B.b_completion[ro + bb[u]];
    }
#pragma unroll
    for (int u = 0; u < kSloUnroll; u++) {
      const int i = i0 + u * kSloThreads + threadIdx.x;
      if (i < n) {
        const double lat = bc[u] - at[u];
        const bool met = lat <= models[S.model_off + mm[u]].slo_ms;
        B.r_slo_met[ro + i] = met;
        const bool in = at[u] >= cutoff;
        if (in) {
          atomicAdd(&cnt_n[mm[u]], 1);
          atomicAdd(&cnt_met[mm[u]], met ? 1 : 0);
        }
        const unsigned long long key = lat_key(lat);
        if (cached) {
          kcache[i] = key;
          mcache[i] = in ? (unsigned char)mm[u] : (unsigned char)255;
        }
        const unsigned hk = (unsigned)(key >> 32);
        kmin = hk < kmin ? hk : kmin;
        kmax = hk > kmax ? hk : kmax;
      }
    }
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (lane == 0 && kmin <= kmax) {
    atomicMin(&hi_min, kmin);
    atomicMax(&hi_max, kmax);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int m = 0; m < S.n_models; m++) tot += cnt_n[m];
    if (tot == 0 && n > 0) use_all = 1;  // `metrics.py:67`: trimmed or records
  }
  __syncthreads();
  if (use_all) {
    __syncthreads();
    for (int m = threadIdx.x; m < kMaxModels; m += blockDim.x) cnt_n[m] = cnt_met[m] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int m = B.arr_model[ro + i];
      atomicAdd(&cnt_n[m], 1);
      atomicAdd(&cnt_met[m], B.r_slo_met[ro + i] ? 1 : 0);
      if (cached) mcache[i] = (unsigned char)m;
    }
    __syncthreads();
  }
  const double cut = use_all ? -INFINITY : cutoff;
  for (int m = threadIdx.x; m < S.n_models; m += blockDim.x) {
    out_n[S.model_off + m] = cnt_n[m];
    out_met[S.model_off + m] = cnt_met[m];
  }
  const double pq[3] = {50.0, 95.0, 99.0};
  const unsigned long long base = n > 0 ? (unsigned long long)hi_min << 32 : 0ull;
  const unsigned span = n > 0 ? hi_max - hi_min : 0u;
  const int T = 32 + (span ? 32 - __clz(span) : 0);  // every v = key - base < 2^T
  for (int g0 = 0; g0 < S.n_models; g0 += kSloGroup) {
    const int gm = min(kSloGroup, S.n_models - g0);
    if (threadIdx.x < gm * 3) {
      const int mm = threadIdx.x / 3, q = threadIdx.x % 3;
      const int nm = cnt_n[g0 + mm];
      // rank = max(1, ceil(p/100 * n)) (`metrics.py:35`)
      int rk = (int)ceil((pq[q] / 100.0) * (double)nm);
      rk = rk < 1 ? 1 : rk;
      rank_left[mm][q] = rk - 1;
      prefix[mm][q] = 0ull;
    }
    if (cached) {  // pass 0's candidates: the group's (trimmed) records
      if (threadIdx.x == 0) n_cand[0] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int m = (int)mcache[i] - g0;
        const bool want = m >= 0 && m < gm;
        const unsigned act = __activemask(), bal = __ballot_sync(act, want);
        const int leader = __ffs(act) - 1;
        int cb = 0;
        if (lane == leader && bal) cb = atomicAdd(&n_cand[0], __popc(bal));
        cb = __shfl_sync(act, cb, leader);
        if (want) cand[0][cb + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)i;
      }
    }
    int pass = 0;
    for (int shift = T - 8; shift > -8; shift -= 8, pass++) {
      const int nq = pass == 0 ? 1 : 3;  // the first pass: one histogram per model (every prefix empty)
      for (int k = threadIdx.x; k < gm * 3 * 256; k += blockDim.x)
        if ((k >> 8) % 3 < nq) (&hist[0][0][0])[k] = 0u;  // rows in use only
      if (threadIdx.x == 0) {
        n_cand[(pass + 1) & 1] = 0;
        unresolved[pass & 1] = 0;
      }
      __syncthreads();
      const unsigned short* cur = cand[pass & 1];
      const int n_iter = cached ? n_cand[pass & 1] : n;
      for (int ii = threadIdx.x; ii < n_iter; ii += blockDim.x) {
        const int i = cached ? (int)cur[ii] : ii;
        int m;
        unsigned long long key;
        if (cached) {
          m = (int)mcache[i] - g0;
          if (m < 0 || m >= gm) continue;  // (255 = trimmed record)
          key = kcache[i];
        } else {
          m = B.arr_model[ro + i] - g0;
          if (m < 0 || m >= gm) continue;
          const double at = B.arr_t[ro + i];
          if (!(at >= cut)) continue;
          key = lat_key(B.b_completion[ro + B.r_batch[ro + i]] - at);
        }
        const unsigned long long v = key - base;
        const unsigned d = slo_digit(v, shift);
        if (pass == 0) {
          atomicAdd(&hist[m][0][d], 1u);
        } else {
#pragma unroll
          for (int q = 0; q < 3; q++)
            if (slo_match(v, prefix[m][q], shift + 8)) atomicAdd(&hist[m][q][d], 1u);
        }
      }
      __syncthreads();
      // digit selection: one warp per (model, quantile), lanes scan 8 bins each
      for (int t = warp; t < gm * 3; t += kSloThreads / 32) {
        const int mm = t / 3, q = t % 3;
        const unsigned int* h = hist[mm][pass == 0 ? 0 : q];
        int c8[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
          c8[j] = (int)h[lane * 8 + j];
          sum += c8[j];
        }
        int incl = sum;  // inclusive scan over lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int excl = incl - sum, left = rank_left[mm][q];
        // the lane whose bins contain rank `left` (the last lane if ranks run out,
        // as the sequential scan stops at digit 255)
        const bool mine = (left >= excl && left < incl) || (lane == 31 && left >= incl);
        const unsigned who = __ballot_sync(0xffffffffu, mine);
        __syncwarp();  // every lane has read rank_left[mm][q] before the owner lane rewrites it
        if (lane == __ffs(who) - 1) {
          int l = left - excl;
          unsigned int d = lane * 8;
          int held = 0;
          for (int j = 0; j < 8; j++, d++) {
            held = c8[j];
            if (d == 255u || l < c8[j]) break;
            l -= c8[j];
          }
          rank_left[mm][q] = l;
          prefix[mm][q] |= slo_put(d, shift);
          if (held > kSloFinish) atomicAdd(&unresolved[pass & 1], 1);
        }
      }
      __syncthreads();
      if (cached && shift > 0) {  // keep the records that still match one of their model's prefixes
        int* nn = &n_cand[(pass + 1) & 1];
        unsigned short* nxt = cand[(pass + 1) & 1];
        for (int ii = threadIdx.x; ii < n_iter; ii += blockDim.x) {
          const int i = (int)cur[ii];
          const int m = (int)mcache[i] - g0;
          const unsigned long long v = kcache[i] - base;
          bool keep = false;
#pragma unroll
          for (int q = 0; q < 3; q++) keep |= slo_match(v, prefix[m][q], shift);
          const unsigned act = __activemask(), bal = __ballot_sync(act, keep);
          const int leader = __ffs(act) - 1;
          int cb = 0;
          if (lane == leader && bal) cb = atomicAdd(nn, __popc(bal));
          cb = __shfl_sync(act, cb, leader);
          if (keep) nxt[cb + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)i;
        }
        __syncthreads();
        if (unresolved[pass & 1] == 0) {
          // every selected bin holds <= kSloFinish records: one warp per
          // (model, quantile) gathers its bin's records and ranks them
          const int nc = n_cand[(pass + 1) & 1];
          for (int t = warp; t < gm * 3; t += kSloThreads / 32) {
            const int mm = t / 3, q = t % 3;
            const unsigned long long pv = prefix[mm][q];
            int c = 0;
            for (int j0 = 0; j0 < nc; j0 += 32) {
              const int j = j0 + lane;
              bool hit = false;
              unsigned long long v = 0ull;
              if (j < nc) {
                const int i = (int)nxt[j];
                v = kcache[i] - base;
                hit = (int)mcache[i] - g0 == mm && slo_match(v, pv, shift);
              }
              const unsigned bal = __ballot_sync(0xffffffffu, hit);
              const int pos = c + __popc(bal & ((1u << lane) - 1u));
              if (hit && pos < kSloFinish) fin[warp][pos] = v;  // (<= kSloFinish hits by construction)
              c += __popc(bal);
            }
            __syncwarp();
            const int want = rank_left[mm][q];
            c = c < kSloFinish ? c : kSloFinish;
            if (lane < c) {
              const unsigned long long x = fin[warp][lane];
              int r = 0;
              for (int k = 0; k < c; k++) {
                const unsigned long long y = fin[warp][k];
                r += (y < x || (y == x && k < lane)) ? 1 : 0;
              }
              if (r == want) prefix[mm][q] = x;
            }
            __syncwarp();
          }
          __syncthreads();
          break;
        }
      }
    }
    if (threadIdx.x < gm * 3) {
      const int mm = threadIdx.x / 3, q = threadIdx.x % 3;
      out_p[3 * (S.model_off + g0 + mm) + q] = cnt_n[g0 + mm] ? key_lat(prefix[mm][q] + base) : NAN;
    }
    __syncthreads();
  }
}

// ---- K3 (large scenarios): the same report with grid-wide passes and global
// histograms, for scenarios too big for one block (long traces, C4).
// ws layout (int32 units): [0,64) n/met with cutoff, [64,128) n/met without,
// [128] use_all, then hist [32][3][256] (u32), prefix [32][3] (u64, 8-aligned),
// left [32][3] (i64).
constexpr int kSloWsHist = 256;
constexpr int kSloWsPrefix = kSloWsHist + kMaxModels * 3 * 256;
constexpr int kSloWsLeft = kSloWsPrefix + kMaxModels * 3 * 2;
constexpr int kSloWsInts = kSloWsLeft + kMaxModels * 3 * 2;
static_assert(kSloWsInts == INTF_SLO_WS_INTS, "slo_ws size mismatch with the header");

// per-request latency keys + model codes for the radix passes of a long
// trace, in the scenario's arrival-list buffers (list_t / list_rid: free once
// the batches are formed); cap = the scenario's list capacity (>= n_req
// unless the lists overflowed -- then the passes gather as before)
constexpr int kSloWarm = 0x100;  // code bit: arrival at or after the warm-up cutoff
struct SloKeys {
  unsigned long long* key;
  int32_t* code;
  long long cap;
};
__device__ __forceinline__ SloKeys slo_keys(const intf_scenario& S, const intf_model* __restrict__ models,
                                            const intf_replay_buffers& B) {
  const intf_model& f = models[S.model_off];
  const intf_model& l = models[S.model_off + S.n_models - 1];
  SloKeys K;
  K.key = reinterpret_cast<unsigned long long*>(B.list_t + f.list_off);
  K.code = B.list_rid + f.list_off;
  K.cap = (long long)l.list_off + l.list_cap - f.list_off;
  return K;
}

// ws scalars after the counters: [129] T, [130] ~(min key high word),
// [131] max key high word (both by atomicMax on the zeroed words), [132]
// state (0 radix passes, 1 every selected bin <= kSloFinish: fetch and rank,
// 2 prefixes complete), [134] the shift the prefixes are complete down to.  In state 1 the histogram region holds
// the fetched bins: counts [96], then [96][kSloFinish] keys (u64).
constexpr int kSloWsT = 129, kSloWsMin = 130, kSloWsMax = 131, kSloWsState = 132,
              kSloWsShift = 134;
constexpr int kSloWsFetchCnt = kSloWsHist, kSloWsFetch = kSloWsHist + kMaxModels * 3;
static_assert(kSloWsFetch % 2 == 0, "fetched keys must be 8-byte aligned");
__device__ __forceinline__ unsigned long long slo_big_base(const int32_t* ws) {
  return (unsigned long long)(~(unsigned)ws[kSloWsMin]) << 32;
}

__global__ void k_slo_big_count(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                                intf_replay_buffers B, int s, const double* __restrict__ warm_cutoff,
                                int32_t* __restrict__ ws) {
  // per-block counters in shared memory, one global atomic per block and
  // counter (10^6 requests onto <= 128 global counters would serialise)
  __shared__ int cnt[128];
  for (int k = threadIdx.x; k < 128; k += blockDim.x) cnt[k] = 0;
  __syncthreads();
  const intf_scenario& S = scen[s];
  const int n = B.n_req[s], ro = S.req_off;
  const double cutoff = warm_cutoff ? warm_cutoff[s] : -INFINITY;
  const SloKeys K = slo_keys(S, models, B);
  unsigned kmin = 0xffffffffu, kmax = 0u;  // key high words: the radix range
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const long long i = i0 + threadIdx.x;
    if (i < n) {
      const int b = B.r_batch[ro + i];
      const double at = B.arr_t[ro + i];
      const int m = B.arr_model[ro + i];
      const double lat = B.b_completion[ro + b] - at;
      const bool met = lat <= models[S.model_off + m].slo_ms;
      B.r_slo_met[ro + i] = met;
      const unsigned long long key = lat_key(lat);
      if (i < K.cap) {  // the radix passes stream these instead of gathering again
        K.key[i] = key;
        K.code[i] = m | (at >= cutoff ? kSloWarm : 0);
      }
      const unsigned hk = (unsigned)(key >> 32);
      kmin = hk < kmin ? hk : kmin;
      kmax = hk > kmax ? hk : kmax;
      // one shared atomic per (model, counter) and warp, not per record
      const unsigned act = __activemask();
      const unsigned same = __match_any_sync(act, m);
      const unsigned bm = __ballot_sync(act, met), bw = __ballot_sync(act, at >= cutoff);
      if ((threadIdx.x & 31) == __ffs(same) - 1) {
        atomicAdd(&cnt[64 + 2 * m], __popc(same));
        atomicAdd(&cnt[64 + 2 * m + 1], __popc(same & bm));
        atomicAdd(&cnt[2 * m], __popc(same & bw));
        atomicAdd(&cnt[2 * m + 1], __popc(same & bw & bm));
      }
    }
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if ((threadIdx.x & 31) == 0 && kmin <= kmax) {
    atomicMax(reinterpret_cast<unsigned*>(ws + kSloWsMin), ~kmin);
    atomicMax(reinterpret_cast<unsigned*>(ws + kSloWsMax), kmax);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 128; k += blockDim.x)
    if (cnt[k]) atomicAdd(&ws[k], cnt[k]);
}

__global__ void k_slo_big_init(const intf_scenario* __restrict__ scen, int s, int32_t* __restrict__ ws,
                               int32_t* out_n, int32_t* out_met) {
  const intf_scenario& S = scen[s];
  __shared__ int use_all;
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int m = 0; m < S.n_models; m++) tot += ws[2 * m];
    int all = 0;
    for (int m = 0; m < S.n_models; m++) all += ws[64 + 2 * m];
    use_all = tot == 0 && all > 0;  // `metrics.py:67`: trimmed or records
    ws[128] = use_all;
    const unsigned lo = ~(unsigned)ws[kSloWsMin], hi = (unsigned)ws[kSloWsMax];
    const unsigned span = all > 0 && hi > lo ? hi - lo : 0u;
    ws[kSloWsT] = 32 + (span ? 32 - __clz(span) : 0);  // every v = key - base < 2^T
    ws[kSloWsState] = 0;
  }
  __syncthreads();
  const double pq[3] = {50.0, 95.0, 99.0};
  unsigned long long* prefix = reinterpret_cast<unsigned long long*>(ws + kSloWsPrefix);
  long long* left = reinterpret_cast<long long*>(ws + kSloWsLeft);
  for (int t = threadIdx.x; t < S.n_models * 3; t += blockDim.x) {
    const int m = t / 3, q = t % 3;
    const int nm = ws[(use_all ? 64 : 0) + 2 * m];
    long long rk = (long long)ceil((pq[q] / 100.0) * (double)nm);
    left[t] = (rk < 1 ? 1 : rk) - 1;
    prefix[t] = 0ull;
    if (q == 0) {
      out_n[S.model_off + m] = nm;
      out_met[S.model_off + m] = ws[(use_all ? 64 : 0) + 2 * m + 1];
    }
  }
  for (int t = threadIdx.x; t < kMaxModels * 3 * 256; t += blockDim.x) ws[kSloWsHist + t] = 0;
}

// radix pass `pass` over v = key - base at digit [T - 8 (pass + 1), + 8);
// the first pass has one histogram per model (every prefix empty)
__global__ void k_slo_big_hist(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                               intf_replay_buffers B, int s, int pass, const double* __restrict__ warm_cutoff,
                               int32_t* __restrict__ ws) {
  if (ws[kSloWsState] != 0) return;  // every (model, quantile) already narrowed
  const int shift = ws[kSloWsT] - 8 * (pass + 1);
  if (shift <= -8) return;
  const intf_scenario& S = scen[s];
  const int n = B.n_req[s], ro = S.req_off;
  const double cutoff = (warm_cutoff && !ws[128]) ? warm_cutoff[s] : -INFINITY;
  const unsigned long long base = slo_big_base(ws);
  const unsigned long long* prefix = reinterpret_cast<const unsigned long long*>(ws + kSloWsPrefix);
  unsigned int* hist = reinterpret_cast<unsigned int*>(ws + kSloWsHist);
  // warp-aggregated increments: latencies of one model share the high key
  // bytes, so most lanes of a warp hit the same bin (one atomic per distinct bin)
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const SloKeys K = slo_keys(S, models, B);
  const bool staged = n <= K.cap;
  const bool all = !(warm_cutoff && !ws[128]);
  const int nq = pass == 0 ? 1 : 3;
  // pass 0 (every in-window record, few hot bins): block-private histogram in
  // shared memory, flushed once (global atomics on the hot bins serialised:
  // 92 us of 1e6 records)
  __shared__ unsigned sh0[kMaxModels * 256];
  if (pass == 0) {
    for (int k = threadIdx.x; k < S.n_models * 256; k += blockDim.x) sh0[k] = 0u;
    __syncthreads();
  }
  for (long long i0 = start - (threadIdx.x & 31); i0 < n; i0 += stride) {
    const long long i = i0 + (threadIdx.x & 31);
    int bins[3] = {-1, -1, -1};
    if (i < n) {
      int m;
      unsigned long long key;
      bool in;
      if (staged) {
        const int c = K.code[i];
        m = c & (kSloWarm - 1);
        in = all || (c & kSloWarm);
        key = K.key[i];
      } else {
        const double at = B.arr_t[ro + i];
        in = at >= cutoff;
        m = B.arr_model[ro + i];
        key = in ? lat_key(B.b_completion[ro + B.r_batch[ro + i]] - at) : 0ull;
      }
      if (in) {
        const unsigned long long v = key - base;
        const int d = (int)slo_digit(v, shift);
        if (pass == 0) {
          bins[0] = m * 256 + d;  // (shared row m)
        } else {
#pragma unroll
          for (int q = 0; q < 3; q++)
            if (slo_match(v, prefix[m * 3 + q], shift + 8)) bins[q] = (m * 3 + q) * 256 + d;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 3; q++) {
      if (q >= nq || !__any_sync(0xffffffffu, bins[q] >= 0)) continue;  // (most records match no prefix)
      const unsigned same = __match_any_sync(0xffffffffu, bins[q]);
      if (bins[q] >= 0 && (threadIdx.x & 31) == __ffs(same) - 1) {
        if (pass == 0) atomicAdd(&sh0[bins[q]], (unsigned)__popc(same));
        else atomicAdd(&hist[bins[q]], (unsigned)__popc(same));
      }
    }
  }
  if (pass == 0) {
    __syncthreads();
    for (int k = threadIdx.x; k < S.n_models * 256; k += blockDim.x)
      if (sh0[k]) atomicAdd(&hist[(k >> 8) * 3 * 256 + (k & 255)], sh0[k]);
  }
}

__global__ void __launch_bounds__(1024) k_slo_big_select(const intf_scenario* __restrict__ scen, int s, int pass,
                                                         int32_t* __restrict__ ws, double* out_p) {
  if (ws[kSloWsState] != 0) return;
  const int shift = ws[kSloWsT] - 8 * (pass + 1);
  if (shift <= -8) return;
  const intf_scenario& S = scen[s];
  unsigned long long* prefix = reinterpret_cast<unsigned long long*>(ws + kSloWsPrefix);
  long long* left = reinterpret_cast<long long*>(ws + kSloWsLeft);
  unsigned int* hist = reinterpret_cast<unsigned int*>(ws + kSloWsHist);
  __shared__ int unres;
  if (threadIdx.x == 0) unres = 0;
  __syncthreads();
  // warp per target (model, percentile): lane owns bins [8 lane, 8 lane + 8);
  // the digit is the first bin whose running count passes `left`
  const int lane = threadIdx.x & 31;
  for (int t = threadIdx.x >> 5; t < S.n_models * 3; t += blockDim.x >> 5) {
    const int row = pass == 0 ? t - t % 3 : t;
    unsigned h[8];
    long long own = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      h[k] = hist[row * 256 + 8 * lane + k];
      own += h[k];
    }
    long long incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long a = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += a;
    }
    const long long l = left[t];
    // the first lane whose inclusive count exceeds l holds the digit (lane 31 if none: digit 255)
    const unsigned hit = __ballot_sync(0xffffffffu, incl > l);
    const int src = hit ? __ffs(hit) - 1 : 31;
    if (lane == src) {
      long long r = l - (incl - own);
      unsigned d = 8u * lane;
      int k = 0;
      for (; k < 7; k++, d++) {
        if (r < (long long)h[k]) break;
        r -= h[k];
      }
      left[t] = r;
      prefix[t] |= slo_put(d, shift);
      if (h[k] > (unsigned)kSloFinish) atomicAdd(&unres, 1);
    }
  }
  __syncthreads();  // every row read: clear for the next pass
  for (int k = threadIdx.x; k < S.n_models * 3 * 256; k += blockDim.x) hist[k] = 0u;
  if (threadIdx.x == 0) {
    if (shift <= 0) {
      ws[kSloWsState] = 2;  // every bit selected: the prefixes are the keys
    } else if (unres == 0) {
      ws[kSloWsState] = 1;  // every selected bin holds <= kSloFinish records: fetch them
      ws[kSloWsShift] = shift;
    }
  }
}

// state 1: the records of every (model, quantile)'s selected bin into the
// (cleared) histogram region, <= kSloFinish each
__global__ void k_slo_big_fetch(const intf_scenario* __restrict__ scen, const intf_model* __restrict__ models,
                                intf_replay_buffers B, int s, const double* __restrict__ warm_cutoff,
                                int32_t* __restrict__ ws) {
  if (ws[kSloWsState] != 1) return;
  const int shift = ws[kSloWsShift];
  const intf_scenario& S = scen[s];
  const int n = B.n_req[s], ro = S.req_off;
  const double cutoff = (warm_cutoff && !ws[128]) ? warm_cutoff[s] : -INFINITY;
  const unsigned long long base = slo_big_base(ws);
  const unsigned long long* prefix = reinterpret_cast<const unsigned long long*>(ws + kSloWsPrefix);
  int* fcnt = ws + kSloWsFetchCnt;
  unsigned long long* fkey = reinterpret_cast<unsigned long long*>(ws + kSloWsFetch);
  const SloKeys K = slo_keys(S, models, B);
  const bool staged = n <= K.cap;
  const bool all = !(warm_cutoff && !ws[128]);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int m;
    unsigned long long key;
    bool in;
    if (staged) {
      const int c = K.code[i];
      m = c & (kSloWarm - 1);
      in = all || (c & kSloWarm);
      key = K.key[i];
    } else {
      const double at = B.arr_t[ro + i];
      in = at >= cutoff;
      m = B.arr_model[ro + i];
      key = in ? lat_key(B.b_completion[ro + B.r_batch[ro + i]] - at) : 0ull;
    }
    if (!in) continue;
    const unsigned long long v = key - base;
#pragma unroll
    for (int q = 0; q < 3; q++) {
      if (slo_match(v, prefix[m * 3 + q], shift)) {
        const int at = atomicAdd(&fcnt[m * 3 + q], 1);
        if (at < kSloFinish) fkey[(m * 3 + q) * kSloFinish + at] = v;
      }
    }
  }
}

// the percentiles: state 1 ranks each fetched bin (one warp per target),
// state 2 reads the complete prefixes
__global__ void __launch_bounds__(1024) k_slo_big_finish(const intf_scenario* __restrict__ scen, int s,
                                                         int32_t* __restrict__ ws, double* out_p) {
  const intf_scenario& S = scen[s];
  const int state = ws[kSloWsState];
  const unsigned long long base = slo_big_base(ws);
  unsigned long long* prefix = reinterpret_cast<unsigned long long*>(ws + kSloWsPrefix);
  const long long* left = reinterpret_cast<const long long*>(ws + kSloWsLeft);
  const int* fcnt = ws + kSloWsFetchCnt;
  const unsigned long long* fkey = reinterpret_cast<const unsigned long long*>(ws + kSloWsFetch);
  const int lane = threadIdx.x & 31;
  for (int t = threadIdx.x >> 5; t < S.n_models * 3; t += blockDim.x >> 5) {
    unsigned long long p = prefix[t];
    if (state == 1) {
      const int c = min(fcnt[t], kSloFinish);
      const unsigned long long x = lane < c ? fkey[t * kSloFinish + lane] : 0ull;
      int r = 0;
      for (int k = 0; k < c; k++) {
        const unsigned long long y = __shfl_sync(0xffffffffu, x, k);
        r += (y < x || (y == x && k < lane)) ? 1 : 0;
      }
      const unsigned win = __ballot_sync(0xffffffffu, lane < c && r == (int)left[t]);
      if (win) p = __shfl_sync(0xffffffffu, x, __ffs(win) - 1);
    }
    if (lane == 0) {
      const int m = t / 3;
      const int nm = ws[(ws[128] ? 64 : 0) + 2 * m];
      out_p[3 * (S.model_off + m) + t % 3] = nm ? key_lat(p + base) : NAN;
    }
  }
}

// ---- K4+K5: features + predictions per outcome; grid (chunks, scenarios).
constexpr int kMaxPred = 8;
struct PredBlock {
  intf_predictor p[kMaxPred];
};

// features + predictions of outcome slot `slot` of scenario S
__device__ __forceinline__ void features_slot(const intf_scenario& S, long long slot,
                                              const intf_model* __restrict__ models, const intf_table& tab,
                                              const intf_replay_buffers& B, const PredBlock& P, int n_pred,
                                              long long slot_stride, double* __restrict__ X, double* __restrict__ Y,
                                              double* __restrict__ Yhat) {
  const int b = B.out_order[slot];
  const long long bslot = (long long)S.req_off + b;
  const int entry = models[S.model_off + B.b_model[bslot]].entry_base + B.b_size[bslot] - 1;
  const double own[3] = {tab.thr[3 * entry], tab.thr[3 * entry + 1], tab.thr[3 * entry + 2]};
  const double* colo = B.s_colo + 3ll * B.b_seg_off[bslot];
  const int nseg = B.b_nseg[bslot];
  Y[slot] = B.b_measured[bslot] / tab.solo_ms[entry];  // interference ratio (`simcore.py:83-85`)
  for (int p = 0; p < n_pred; p++) {
    double x[6];
    features_one(own, colo, nseg, P.p[p].ewma, P.p[p].alpha, x);
    if (X) {
      double* xo = X + (p * slot_stride + slot) * 6;
#pragma unroll
      for (int i = 0; i < 6; i++) xo[i] = x[i];
    }
    Yhat[p * slot_stride + slot] = predict7(P.p[p].w, x);
  }
}

// thread per outcome; launch shape as k_noise_table (block per scenario for
// many scenarios, grid-stride over packed slots for few long ones)
__global__ void k_features(const intf_scenario* __restrict__ scen, int n_scen, long long req_slots,
                           const intf_model* __restrict__ models, intf_table tab, intf_replay_buffers B, PredBlock P,
                           int n_pred, long long slot_stride, double* __restrict__ X, double* __restrict__ Y,
                           double* __restrict__ Yhat) {
  if (n_scen >= kPerScenarioMin) {
    for (int s = blockIdx.x; s < n_scen; s += gridDim.x) {
      const intf_scenario& S = scen[s];
      const int nb = B.n_batches[s];
      for (int k = threadIdx.x; k < nb; k += blockDim.x)
        features_slot(S, (long long)S.req_off + k, models, tab, B, P, n_pred, slot_stride, X, Y, Yhat);
    }
    return;
  }
  for (long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x; slot < req_slots;
       slot += (long long)gridDim.x * blockDim.x) {
    const int s = scen_of_slot(scen, n_scen, slot);
    if (slot - scen[s].req_off < B.n_batches[s])
      features_slot(scen[s], slot, models, tab, B, P, n_pred, slot_stride, X, Y, Yhat);
  }
}

// Longest-first order of a long trace's todo list: a counting sort by
// batches per job, descending (the jobs kernel takes the list in order, so
// the longest jobs start first instead of wherever the plan placed them:
// C4 pass 1 0.72 -> 0.6 ms).  Scratch: jobs->scratch (free after the plan).
constexpr int kLptBuckets = kOrderBuckets;
__device__ __forceinline__ int lpt_bucket(const intf_jobs& J, int slot) {
  const int len = J.hi[slot] - J.lo[slot];
  return kLptBuckets - 1 - (len < 0 ? 0 : (len < kLptBuckets - 1 ? len : kLptBuckets - 1));
}
__global__ void k_todo_lpt_hist(intf_jobs J, int32_t* __restrict__ cnt) {
  const int n = *J.todo_count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&cnt[lpt_bucket(J, J.todo[i])], 1);
}
__global__ void k_todo_lpt_scatter(intf_jobs J, int32_t* __restrict__ cnt, int32_t* __restrict__ tmp) {
  const int n = *J.todo_count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int sl = J.todo[i];
    tmp[atomicAdd(&cnt[lpt_bucket(J, sl)], 1)] = sl;
  }
}
__global__ void k_todo_copy(intf_jobs J, const int32_t* __restrict__ tmp) {
  const int n = *J.todo_count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) J.todo[i] = tmp[i];
}
int todo_lpt(const intf_jobs* jobs, cudaStream_t st) {
  int32_t* cnt = reinterpret_cast<int32_t*>(jobs->scratch);
  int32_t* tmp = cnt + kLptBuckets;
  if (12ll * jobs->total_slots < kLptBuckets + (long long)jobs->total_slots) return INTF_OK;  // (tiny: keep the order)
  cudaMemsetAsync(cnt, 0, sizeof(int32_t) * kLptBuckets, st);
  k_todo_lpt_hist<<<148 * 4, 256, 0, st>>>(*jobs, cnt);
  k_order_scan<<<1, 1024, 0, st>>>(cnt);
  k_todo_lpt_scatter<<<148 * 4, 256, 0, st>>>(*jobs, cnt, tmp);
  k_todo_copy<<<148 * 4, 256, 0, st>>>(*jobs, tmp);
  return launch_status("k_todo_lpt");
}

unsigned noise_grid(const intf_batch* bt, int K) {
  (void)K;
  if (bt->n_scen >= kPerScenarioMin) return bt->n_scen < 65535 ? bt->n_scen : 65535;
  const long long n = (long long)bt->req_slots;  // (a thread per batch slot)
  const long long blocks = (n + 255) / 256;
  return (unsigned)(blocks < 148 * 16 ? (blocks > 0 ? blocks : 1) : 148 * 16);
}

// (element chunks, models): enough blocks per model list that long traces use
// every SM, one block per model for short ones; models beyond 65535 spill into z
dim3 merge_grid(const intf_batch* bt) {
  const long long per_model = bt->max_list_cap > 0 ? bt->max_list_cap : 1;
  unsigned x = ceil_div(per_model, 256 * 4);
  const unsigned m = bt->n_models > 0 ? (unsigned)bt->n_models : 1u;
  const unsigned y = m < 65535u ? m : 65535u;
  return dim3(x < 1 ? 1 : x, y, ceil_div(m, y));
}

int launch_formation(const intf_batch* bt, const intf_replay_buffers* buf, cudaStream_t st) {
  if (!buf->mb_t || !buf->mb_info || !buf->n_mb) return bad_input("formation scratch (mb_t, mb_info, n_mb) missing");
  int rc;
  cudaMemsetAsync(buf->n_batches, 0, sizeof(int32_t) * bt->n_scen, st);
  k_form_status<<<ceil_div(bt->n_scen, 128), 128, 0, st>>>(bt->scen, bt->n_scen, *buf);
  if ((rc = launch_status("k_form_status"))) return rc;
  if (bt->n_models <= 0) return INTF_OK;
  k_form_models<<<ceil_div(bt->n_models, kFormModelWarps), 32 * kFormModelWarps, 0, st>>>(bt->scen, bt->models,
                                                                                         bt->n_models, *buf);
  if ((rc = launch_status("k_form_models"))) return rc;
  if (bt->max_list_cap >= kLongForm) {  // long model lists: chunked formation
    if (!buf->form_ws) return bad_input("formation of long lists needs form_ws scratch");
    const unsigned m = (unsigned)bt->n_models, y = m < 65535u ? m : 65535u;
    // flat grid over the long lists' 256-entry chunks when the caller gave the map
    const int32_t* blk = bt->long_blocks && bt->n_long_blocks > 0 ? bt->long_blocks : nullptr;
    const dim3 grid = blk ? dim3((unsigned)bt->n_long_blocks) : dim3(ceil_div(bt->max_list_cap, 256), y, ceil_div(m, y));
    k_form_nxt<<<grid, 256, 0, st>>>(bt->scen, bt->models, bt->n_models, *buf, blk);
    if ((rc = launch_status("k_form_nxt"))) return rc;
    const dim3 cgrid(ceil_div(bt->max_list_cap, kFormChunk), y, ceil_div(m, y));
    k_form_chunks<<<cgrid, kFormChunkThreads, 0, st>>>(bt->scen, bt->models, bt->n_models, *buf);
    if ((rc = launch_status("k_form_chunks"))) return rc;
    k_form_compose<<<ceil_div(bt->n_models, 128), 128, 0, st>>>(bt->scen, bt->models, bt->n_models, *buf);
    if ((rc = launch_status("k_form_compose"))) return rc;
    k_form_emit_chunks<<<cgrid, kFormChunkThreads, 0, st>>>(bt->scen, bt->models, bt->n_models, *buf);
    if ((rc = launch_status("k_form_emit_chunks"))) return rc;
  }
  if (bt->max_list_cap < kLongForm) {  // short lists: one warp per model
    k_merge_batches_warp<<<ceil_div(bt->n_models, kMergeWarps), 32 * kMergeWarps, 0, st>>>(bt->scen, bt->models,
                                                                                          *buf, bt->n_models);
    return launch_status("k_merge_batches_warp");
  }
  if (buf->form_ws && bt->n_scen <= 65535 && bt->max_list_cap < (1 << 24)) {
    // long traces: time buckets (form_ws is free after the emit; members packed as model << 24 | index)
    const dim3 g = merge_grid(bt);
    const dim3 tiles(ceil_div(bt->max_req_cap / kArrBucketAvg * 2 + 1, kArrTile), bt->n_scen);
    k_arr_zero<<<tiles, 1024, 0, st>>>(bt->scen, bt->models, *buf);
    k_bat_hist<<<g, 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
    k_arr_scan_tiles<<<tiles, 1024, 0, st>>>(bt->scen, bt->models, *buf);
    k_arr_scan_top<<<ceil_div(bt->n_scen, 128), 128, 0, st>>>(bt->scen, bt->n_scen, bt->models, *buf);
    k_bat_scatter<<<g, 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
    k_bat_place<<<g, 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
    return launch_status("k_bat_place");
  }
  k_merge_batches<<<merge_grid(bt), 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
  return launch_status("k_merge_batches");
}

}  // namespace

extern "C" {

int intf_long_list(void) { return kLongForm; }

int intf_generate_arrivals(const intf_batch* bt, const intf_replay_buffers* buf, void* stream) {
  INTF_RANGE("intf_generate_arrivals");
  if (!bt || !bt->scen || !bt->models || !buf || bt->n_scen <= 0) return bad_input("intf_generate_arrivals: null argument");
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(buf->n_req, 0, sizeof(int32_t) * bt->n_scen, st);
  cudaMemsetAsync(buf->status, 0, sizeof(int32_t) * bt->n_scen, st);
  if (bt->n_models <= 0) return INTF_OK;
  int rc;
  k_gen_arrivals<<<ceil_div(bt->n_models, kGenWarps), 32 * kGenWarps, 0, st>>>(bt->scen, bt->models, bt->n_models,
                                                                               *buf);
  if ((rc = launch_status("k_gen_arrivals"))) return rc;
  if (bt->max_list_cap >= kBigList) {  // long model streams (the warp kernel skipped them)
    const unsigned m = (unsigned)bt->n_models, y = m < 65535u ? m : 65535u;
    k_gen_gaps<<<dim3(ceil_div(bt->max_list_cap, 256 * kGapRun), y, ceil_div(m, y)), 256, 0, st>>>(
        bt->scen, bt->models, bt->n_models, *buf);
    if ((rc = launch_status("k_gen_gaps"))) return rc;
#if INTF_SCAN_SEQ
    k_scan_gaps<<<bt->n_models, 32, 0, st>>>(bt->scen, bt->models, bt->n_models, *buf);
    if ((rc = launch_status("k_scan_gaps"))) return rc;
#else
    const dim3 cgrid(ceil_div(ceil_div(bt->max_list_cap, kScanChunk), 32 * kBinWarps), y, ceil_div(m, y));
    k_bin_sums<<<cgrid, 32 * kBinWarps, 0, st>>>(bt->models, bt->n_models, *buf);
    k_bin_scan<<<bt->n_models, kBinThreads, 0, st>>>(bt->models, bt->n_models, *buf);
    k_bin_classify<<<cgrid, 32 * kBinWarps, 0, st>>>(bt->models, bt->n_models, *buf);
    k_bin_runs<<<bt->n_models, kBinThreads, 0, st>>>(bt->models, bt->n_models, *buf);
    k_bin_fill<<<dim3(ceil_div(ceil_div(bt->max_list_cap, kScanChunk), 128), y, ceil_div(m, y)), 128, 0, st>>>(
        bt->models, bt->n_models, *buf);
    if ((rc = launch_status("k_bin_*"))) return rc;
#endif
    k_fill_gaps<<<dim3(ceil_div(ceil_div(bt->max_list_cap, kScanChunk), 128), y, ceil_div(m, y)), 128, 0, st>>>(
        bt->scen, bt->models, bt->n_models, *buf);
    if ((rc = launch_status("k_fill_gaps"))) return rc;
  }
  if (bt->n_scen >= kPerScenarioMin && bt->max_list_cap < kLongForm) {  // sweeps of short scenarios
    k_merge_arrivals_scen<<<bt->n_scen < 65535 ? bt->n_scen : 65535, 256, 0, st>>>(bt->scen, bt->n_scen, bt->models,
                                                                                 *buf);
    return launch_status("k_merge_arrivals_scen");
  }
  if (buf->form_ws && bt->max_list_cap >= kLongForm && bt->max_list_cap < (1 << 24) && bt->n_scen <= 65535) {
    // long traces: time buckets (members packed as model << 24 | index)
    const dim3 g = merge_grid(bt);
    const dim3 tiles(ceil_div(bt->max_req_cap / kArrBucketAvg * 2 + 1, kArrTile), bt->n_scen);
    k_arr_zero<<<tiles, 1024, 0, st>>>(bt->scen, bt->models, *buf);
    k_arr_hist<<<g, 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
    k_arr_scan_tiles<<<tiles, 1024, 0, st>>>(bt->scen, bt->models, *buf);
    k_arr_scan_top<<<ceil_div(bt->n_scen, 128), 128, 0, st>>>(bt->scen, bt->n_scen, bt->models, *buf);
    k_arr_scatter<<<g, 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
    k_arr_place<<<g, 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
    return launch_status("k_arr_place");
  }
  k_merge_arrivals<<<merge_grid(bt), 256, 0, st>>>(bt->scen, bt->models, *buf, bt->n_models);
  return launch_status("k_merge_arrivals");
}

int intf_split_arrivals(const intf_batch* bt, const intf_replay_buffers* buf, void* stream) {
  INTF_RANGE("intf_split_arrivals");
  if (!bt || !bt->scen || !bt->models || !buf || bt->n_scen <= 0) return bad_input("intf_split_arrivals: null argument");
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(buf->status, 0, sizeof(int32_t) * bt->n_scen, st);
  k_split_arrivals<<<ceil_div(bt->n_scen, 64), 64, 0, st>>>(bt->scen, bt->n_scen, bt->models, *buf);
  return launch_status("k_split_arrivals");
}

int intf_form_batches(const intf_batch* bt, const intf_replay_buffers* buf, void* stream) {
  INTF_RANGE("intf_form_batches");
  if (!bt || !bt->scen || !bt->models || !buf || bt->n_scen <= 0) return bad_input("intf_form_batches: null argument");
  if (buf->noise_k > 0 && !buf->noise_tab) return bad_input("intf_form_batches: noise_k > 0 needs noise_tab");
  cudaStream_t st = as_stream(stream);
  int rc;
  if ((rc = launch_formation(bt, buf, st))) return rc;
  if (buf->noise_k > 0 && bt->max_req_cap > 0) {
    k_noise_table<<<noise_grid(bt, buf->noise_k), 256, 0, st>>>(bt->scen, bt->n_scen, (long long)bt->req_slots,
                                                                 *buf);
    if ((rc = launch_status("k_noise_table"))) return rc;
  }
  return INTF_OK;
}

int intf_replay_jobs(const intf_batch* bt, const intf_table* table, const intf_replay_buffers* buf,
                     const int32_t* job_scen, const int32_t* job_lo, const int32_t* job_hi, int32_t n_jobs,
                     double* job_last_done, int32_t* job_info, void* stream) {
  INTF_RANGE("intf_replay_jobs");
  if (!bt || !bt->scen || !bt->models || !buf || !table || !job_scen || !job_lo || !job_hi || !job_last_done ||
      !job_info || n_jobs < 0)
    return bad_input("intf_replay_jobs: null argument");
  if (buf->cap_max > kMaxCap || buf->cap_max < 1 || buf->seg_stride < 1)
    return bad_input("intf_replay_jobs: cap_max must be in [1, 8], seg_stride >= 1");
  if (n_jobs == 0) return INTF_OK;
  k_replay_jobs<<<ceil_div(n_jobs, kJobWarps * (32 / kReplayW)), 32 * kJobWarps, 0, as_stream(stream)>>>(
      bt->scen, bt->models, *table, *buf, job_scen, job_lo, job_hi, n_jobs, job_last_done, job_info);
  return launch_status("k_replay_jobs");
}

int intf_jobs_plan(const intf_batch* bt, const intf_table* table, const intf_replay_buffers* buf, const intf_jobs* jobs,
                   void* stream) {
  INTF_RANGE("intf_jobs_plan");
  if (!bt || !bt->scen || !table || !buf || !jobs || !jobs->todo_count || jobs->min_len < 1)
    return bad_input("intf_jobs_plan: bad argument");
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(jobs->todo_count, 0, sizeof(int32_t), st);
  k_jobs_plan<<<ceil_div(bt->n_scen, 4), 128, 0, st>>>(bt->scen, bt->n_scen, bt->models, *table, *buf, *jobs);
  int rc = launch_status("k_jobs_plan");
  if (rc || bt->max_req_cap < kBigJobs) return rc;
  if (!jobs->scratch) return bad_input("intf_jobs_plan: long traces need jobs->scratch");
  if (bt->n_scen > 65535 || jobs->min_len > 8192) {  // one block per long scenario
    k_jobs_plan_big<<<bt->n_scen, kBigThreads, 0, st>>>(bt->scen, bt->models, *table, *buf, *jobs);
    if ((rc = launch_status("k_jobs_plan_big"))) return rc;
    return todo_lpt(jobs, st);
  }
  const dim3 grid(ceil_div(bt->max_req_cap, kPlanChunk), bt->n_scen);
  k_plan_p1<<<grid, 256, 0, st>>>(bt->scen, bt->models, *table, *buf, *jobs);
  if ((rc = launch_status("k_plan_p1"))) return rc;
  k_plan_p2<<<bt->n_scen, kBigThreads, 0, st>>>(bt->scen, *buf, *jobs);
  if ((rc = launch_status("k_plan_p2"))) return rc;
  k_plan_p3<<<grid, 256, 0, st>>>(bt->scen, bt->models, *table, *buf, *jobs);
  if ((rc = launch_status("k_plan_p3"))) return rc;
  k_plan_p4<<<bt->n_scen, kBigThreads, 0, st>>>(bt->scen, *buf, *jobs);
  if ((rc = launch_status("k_plan_p4"))) return rc;
  return todo_lpt(jobs, st);
}

int intf_jobs_replay(const intf_batch* bt, const intf_table* table, const intf_replay_buffers* buf,
                     const intf_jobs* jobs, int32_t n_todo, void* stream) {
  INTF_RANGE("intf_jobs_replay");
  if (!bt || !bt->scen || !table || !buf || !jobs || (n_todo < 0 && !jobs->todo_count))
    return bad_input("intf_jobs_replay: bad argument");
  if (buf->cap_max > kMaxCap || buf->cap_max < 1 || buf->seg_stride < 1)
    return bad_input("intf_jobs_replay: cap_max must be in [1, 8], seg_stride >= 1");
  if (n_todo == 0) return INTF_OK;
  // n_todo < 0: up to -n_todo jobs, the count read on the device; a grid of
  // at most one wave, its warps striding over the todo list
  const long long want = ceil_div(n_todo > 0 ? n_todo : -(long long)n_todo, kJobWarps * (32 / kReplayW));
  const unsigned grid = n_todo > 0 ? (unsigned)want : (unsigned)(want < 148 * INTF_JOB_MINB ? want : 148 * INTF_JOB_MINB);
  if (n_todo < 0) cudaMemsetAsync(jobs->todo_count + 1, 0, sizeof(int32_t), as_stream(stream));  // the work counter
  k_jobs_replay<<<grid, 32 * kJobWarps, 0, as_stream(stream)>>>(bt->scen, bt->models, *table, *buf, *jobs, n_todo);
  return launch_status("k_jobs_replay");
}

int intf_jobs_verify(const intf_batch* bt, const intf_replay_buffers* buf, const intf_jobs* jobs, void* stream) {
  INTF_RANGE("intf_jobs_verify");
  if (!bt || !bt->scen || !buf || !jobs || !jobs->todo_count) return bad_input("intf_jobs_verify: bad argument");
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(jobs->todo_count, 0, sizeof(int32_t), st);
  k_jobs_verify<<<ceil_div(bt->n_scen, 128), 128, 0, st>>>(bt->scen, bt->n_scen, *buf, *jobs);
  int rc = launch_status("k_jobs_verify");
  if (rc || bt->max_req_cap < kBigJobs) return rc;
  if (!jobs->scratch) return bad_input("intf_jobs_verify: long traces need jobs->scratch");
  k_jobs_verify_big<<<bt->n_scen, kVerThreads, 0, st>>>(bt->scen, *buf, *jobs);
  return launch_status("k_jobs_verify_big");
}

int intf_replay(const intf_batch* bt, const intf_table* table, const intf_replay_buffers* buf, void* stream) {
  INTF_RANGE("intf_replay");
  if (!bt || !bt->scen || !bt->models || !buf || !table || bt->n_scen <= 0) return bad_input("intf_replay: null argument");
  if (buf->cap_max > kMaxCap || buf->cap_max < 1 || buf->seg_stride < 1 || buf->noise_k < 0)
    return bad_input("intf_replay: cap_max must be in [1, 8], seg_stride >= 1, noise_k >= 0");
  if (buf->noise_k > 0 && !buf->noise_tab) return bad_input("intf_replay: noise_k > 0 needs noise_tab");
  cudaStream_t st = as_stream(stream);
  int rc;
  if ((rc = launch_formation(bt, buf, st))) return rc;
  if (buf->noise_k > 0 && bt->max_req_cap > 0) {
    k_noise_table<<<noise_grid(bt, buf->noise_k), 256, 0, st>>>(bt->scen, bt->n_scen, (long long)bt->req_slots,
                                                                 *buf);
    if ((rc = launch_status("k_noise_table"))) return rc;
  }
  if (!buf->slo_ws || !buf->order) return bad_input("intf_replay: slo_ws / order scratch missing");
  // LPT order via slo_ws (free until the SLO pass): [0] work counter, [1, 1 + 4096) bucket counts
  int32_t* cnt = buf->slo_ws + 1;
  cudaMemsetAsync(buf->slo_ws, 0, sizeof(int32_t) * (1 + kOrderBuckets), st);
  k_order_hist<<<ceil_div(bt->n_scen, 256), 256, 0, st>>>(bt->scen, bt->n_scen, *buf, cnt);
  k_order_scan<<<1, 1024, 0, st>>>(cnt);
  k_order_scatter<<<ceil_div(bt->n_scen, 256), 256, 0, st>>>(bt->scen, bt->n_scen, *buf, cnt);
  if ((rc = launch_status("k_order_*"))) return rc;
  const unsigned per_wave = 148u * INTF_REPLAY_MINB, need = ceil_div(bt->n_scen, kReplayWarps * (32 / kReplayW));
  k_replay_warp<<<need < per_wave ? need : per_wave, 32 * kReplayWarps, 0, st>>>(bt->scen, bt->n_scen, bt->models,
                                                                                  *table, *buf);
  return launch_status("k_replay_warp");
}

int intf_slo_report(const intf_batch* bt, const intf_replay_buffers* buf, const double* warm_cutoff, int32_t* out_n,
                    int32_t* out_met, double* out_p, void* stream) {
  INTF_RANGE("intf_slo_report");
  if (!bt || !bt->scen || !bt->models || !buf || !out_n || !out_met || !out_p || bt->n_scen <= 0)
    return bad_input("intf_slo_report: null argument");
  if (bt->max_req_cap > kSloBigReq) {  // long traces: grid-wide passes, one scenario at a time
    if (!buf->slo_ws) return bad_input("intf_slo_report: large scenarios need slo_ws");
    if (bt->max_models > kMaxModels) return bad_input("intf_slo_report: more than 32 models");
    cudaStream_t st = as_stream(stream);
    int rc;
    for (int s = 0; s < bt->n_scen; s++) {
      cudaMemsetAsync(buf->slo_ws, 0, sizeof(int32_t) * 256, st);
      k_slo_big_count<<<4 * 148, 256, 0, st>>>(bt->scen, bt->models, *buf, s, warm_cutoff, buf->slo_ws);
      if ((rc = launch_status("k_slo_big_count"))) return rc;
      k_slo_big_init<<<1, 256, 0, st>>>(bt->scen, s, buf->slo_ws, out_n, out_met);
      if ((rc = launch_status("k_slo_big_init"))) return rc;
      // <= 8 radix passes (v < 2^64); once every selected bin is small the
      // remaining ones return at once and the bins are fetched and ranked
      for (int pass = 0; pass < 8; pass++) {
        k_slo_big_hist<<<4 * 148, 256, 0, st>>>(bt->scen, bt->models, *buf, s, pass, warm_cutoff, buf->slo_ws);
        k_slo_big_select<<<1, 1024, 0, st>>>(bt->scen, s, pass, buf->slo_ws, out_p);
      }
      if ((rc = launch_status("k_slo_big_select"))) return rc;
      k_slo_big_fetch<<<4 * 148, 256, 0, st>>>(bt->scen, bt->models, *buf, s, warm_cutoff, buf->slo_ws);
      k_slo_big_finish<<<1, 1024, 0, st>>>(bt->scen, s, buf->slo_ws, out_p);
      if ((rc = launch_status("k_slo_big_finish"))) return rc;
    }
    return INTF_OK;
  }
  // keys (8 B) + model ids (1 B): 36 KB dynamic on top of ~25 KB static -> opt-in
  // attribute, set once per device (setting it twice is harmless)
  const size_t smem = (size_t)kSloCache * (9 + 4);  // keys + model ids + two candidate index lists
  int dev = 0;
  cudaGetDevice(&dev);
  static bool attr_set[64] = {};
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaFuncSetAttribute(k_slo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  k_slo<<<bt->n_scen, kSloThreads, smem, as_stream(stream)>>>(bt->scen, bt->models, *buf, warm_cutoff, out_n, out_met,
                                                             out_p);
  return launch_status("k_slo");
}

int intf_features_predict(const intf_batch* bt, const intf_table* table, const intf_replay_buffers* buf,
                          const intf_predictor* preds, int32_t n_pred, int64_t slot_stride, double* X, double* y,
                          double* yhat, void* stream) {
  INTF_RANGE("intf_features_predict");
  if (!bt || !bt->scen || !bt->models || !buf || !table || !y || (n_pred && !yhat) || bt->n_scen <= 0)
    return bad_input("intf_features_predict: bad argument");
  if (n_pred < 0 || n_pred > kMaxPred || (n_pred && !preds)) return bad_input("intf_features_predict: n_pred in [0,8]");
  PredBlock P;
  memset(&P, 0, sizeof(P));
  for (int i = 0; i < n_pred; i++) P.p[i] = preds[i];
  if (bt->max_req_cap <= 0) return INTF_OK;
  const long long blocks = ((long long)bt->req_slots + 127) / 128;
  const unsigned grid = bt->n_scen >= kPerScenarioMin ? (bt->n_scen < 65535 ? bt->n_scen : 65535)
                                                      : (unsigned)(blocks < 148 * 32 ? (blocks > 0 ? blocks : 1) : 148 * 32);
  k_features<<<grid, 128, 0, as_stream(stream)>>>(
      bt->scen, bt->n_scen, (long long)bt->req_slots, bt->models, *table, *buf, P, n_pred, (long long)slot_stride, X,
      y, yhat);
  return launch_status("k_features");
}

}  // extern "C"
