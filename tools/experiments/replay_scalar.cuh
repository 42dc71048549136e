// EXPERIMENT (not built into the product; kept for the record).
// A thread-per-scenario form of the replay with the running set in registers.
// Bit-exact on every golden scenario (all 45 GPU parity tests passed with it
// wired in as k_replay_scalar), but slower on B200 than the warp form:
// C5 at 10^4 scenarios 16.9 ms (1 scenario/warp) .. 19.5 ms (32/warp) vs
// 7.6 ms; the longest cap-2 scenario alone 6.8 ms vs 5.6 ms.  ncu: ~1,110
// SASS instructions per batch (CAPM-way unrolled selects) vs ~810, at the
// same ~5 cycles per dependent instruction.
// replay_scalar.cuh -- the replay recurrence with one THREAD per scenario and
// the running set held in registers (sm_100a).
//
// Same events, arithmetic and outputs as replay_formed() (replay_core.cuh, the
// readable statement) and replay_group() (replay_warp.cuh, a warp per
// scenario, lane = running slot).  The warp form spends most of each event on
// warp-collective bookkeeping (shuffles, ballots, reconvergence) around a
// scalar dependency chain; here the chain runs in one thread:
//   * the running set is a register array of physical slots (a batch keeps
//     its slot while it runs), with a dispatch counter for running-list
//     order;
//   * every slot field is accessed with compile-time indices only (CAPM-way
//     unrolled selects), so nothing spills to local memory;
//   * the next batch to dispatch (model, size, profile row, first noise
//     draws) and the next formation time are prefetched one step ahead, so no
//     global load sits on the chain;
//   * each running batch's open segment history lives in shared memory
//     (kSmemSeg records, global scratch beyond), copied out at completion.
// SPW scenarios share a warp (lane l < SPW runs one scenario each).
#pragma once
#include "replay_warp.cuh"

namespace intf {

constexpr int kScalarNz = 4;  // noise draws held in registers per running batch

template <int CAPM>
struct ScalarSlots {
  double start[CAPM], total[CAPM], progress[CAPM], done[CAPM], own0[CAPM], own1[CAPM], own2[CAPM];
  double tb[CAPM], sd[CAPM], nz[CAPM][kScalarNz];
  int batch[CAPM], nseg[CAPM], non1[CAPM], seq[CAPM];
};

// prefetched description of the next batch to dispatch
struct NextBatch {
  double total, own0, own1, own2, nz[kScalarNz];
  int b;
};

// Slots are physical (a batch keeps its slot, and its shared-memory segment
// history, for its lifetime); `seq` = dispatch counter gives the running-list
// order.  The colo sum of a batch adds its peers' throughputs in running-list
// order from 0; with at most two peers the order cannot change the result
// ((0 + a) + b == (0 + b) + a), so only a full cap-4 set sorts by seq.
template <int CAPM>
__device__ __forceinline__ ReplayJobOut replay_scalar(const ReplayJob J, const intf_scenario& S,
                                                      const intf_model* __restrict__ md, const intf_table tab,
                                                      const intf_replay_buffers B, double* __restrict__ hist,
                                                      int status) {
  const int cap = S.cap, nb = J.b_hi, ro = S.req_off;
  const int K = B.noise_k < kScalarNz ? B.noise_k : kScalarNz;
  const double be[3] = {S.beta[0], S.beta[1], S.beta[2]};
  const double sigma = S.sigma;
  double* gseg = B.slot_seg + (size_t)J.scratch * B.cap_max * (size_t)B.seg_stride * 5;  // [slot][k][5]

  ScalarSlots<CAPM> R;
#pragma unroll
  for (int k = 0; k < CAPM; k++) {
    R.start[k] = R.total[k] = R.progress[k] = R.done[k] = 0.0;
    R.own0[k] = R.own1[k] = R.own2[k] = R.tb[k] = 0.0;
    R.sd[k] = 1.0;
#pragma unroll
    for (int q = 0; q < kScalarNz; q++) R.nz[k][q] = 1.0;
    R.batch[k] = R.nseg[k] = R.non1[k] = R.seq[k] = 0;
  }
  unsigned actm = 0u;  // running slots
  int nrun = 0, seqc = 0;
  double now = 0.0, last_done = -INFINITY;
  int n_formed = J.b_lo, dq = J.b_lo, n_done = J.b_lo, seg_cursor = 0, n_reseats = 0;

  auto fetch_next = [&](int b, NextBatch& nx) {
    nx.b = b;
    if (b < nb) {
      const int entry = md[B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1;
      nx.total = tab.solo_ms[entry];
      nx.own0 = tab.thr[3 * entry];
      nx.own1 = tab.thr[3 * entry + 1];
      nx.own2 = tab.thr[3 * entry + 2];
      const double* nt = B.noise_tab + (size_t)(ro + b) * B.noise_k;
#pragma unroll
      for (int q = 0; q < kScalarNz; q++) nx.nz[q] = q < K ? nt[q] : 1.0;
    }
  };
  NextBatch nx;
  fetch_next(dq, nx);
  double tf_next = n_formed < nb ? B.b_formed[ro + n_formed] : INFINITY;

  auto rec = [&](int h, int k) -> double* {
    return k < kSmemSeg ? hist + (h * kSmemSeg + k) * 5 : gseg + ((size_t)h * B.seg_stride + k) * 5;
  };

  // GpuState._reseat (`simcore.py:133-141`) of slot i (compile-time index)
  auto reseat = [&](const int i) {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    if (CAPM < 4 || nrun < 4) {
#pragma unroll
      for (int q = 0; q < CAPM; q++) {
        if (q != i && ((actm >> q) & 1u)) {
          c0 = c0 + R.own0[q];
          c1 = c1 + R.own1[q];
          c2 = c2 + R.own2[q];
        }
      }
    } else {  // three peers: add in dispatch (seq) order
#pragma unroll
      for (int r = 0; r < CAPM - 1; r++) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int q = 0; q < CAPM; q++) {
          if (q == i) continue;
          int rk = 0;
#pragma unroll
          for (int u = 0; u < CAPM; u++)
            if (u != i && u != q && R.seq[u] < R.seq[q]) rk++;
          if (rk == r) {
            a0 = R.own0[q];
            a1 = R.own1[q];
            a2 = R.own2[q];
          }
        }
        c0 = c0 + a0;
        c1 = c1 + a1;
        c2 = c2 + a2;
      }
    }
    const int ns = R.nseg[i];
    double noise = R.nz[i][0];
#pragma unroll
    for (int q = 1; q < kScalarNz; q++) noise = ns == q ? R.nz[i][q] : noise;
    if (ns >= K) {
      noise = ns < B.noise_k ? B.noise_tab[(size_t)(ro + R.batch[i]) * B.noise_k + ns]
                             : noise_draw_slow(S.oracle_seed, S.batch_id_base + (uint64_t)R.batch[i], (uint64_t)ns,
                                               sigma);
    }
    const double o[3] = {R.own0[i], R.own1[i], R.own2[i]}, colo[3] = {c0, c1, c2};
    const double sd = slowdown(o, colo, be, noise);
    if (ns < B.seg_stride) {
      double* p = rec(i, ns);
      p[0] = now;
      p[1] = sd;
      p[2] = c0;
      p[3] = c1;
      p[4] = c2;
    } else {
      status |= INTF_ST_SEG_STRIDE;
    }
    R.nseg[i] = ns + 1;
    R.tb[i] = now;
    R.sd[i] = sd;
    R.non1[i] += sd != 1.0 ? 1 : 0;
    const double d = now + (R.total[i] - R.progress[i]) * sd;
    R.done[i] = d;
    if (d < now - 1e-9) status |= INTF_ST_PAST_EVENT;
  };
  // RunningBatch.close_segment (`simcore.py:56-66`) of slot i
  auto close = [&](const int i) {
    if (now == R.tb[i]) {  // zero-length: pop, reuse the noise index
      R.nseg[i] -= 1;
      R.non1[i] -= R.sd[i] != 1.0 ? 1 : 0;
    } else {
      R.progress[i] = R.progress[i] + (now - R.tb[i]) / R.sd[i];
    }
  };

  for (;;) {
    // next completion: lexicographic min of (done, batch) over the running set
    double dmin = INFINITY;
    int bmin = 0x7fffffff, ci = 0;
#pragma unroll
    for (int k = 0; k < CAPM; k++) {
      if (((actm >> k) & 1u) && (R.done[k] < dmin || (R.done[k] == dmin && R.batch[k] < bmin))) {
        dmin = R.done[k];
        bmin = R.batch[k];
        ci = k;
      }
    }
    const bool have_form = n_formed < nb;
    if (nrun == 0 && !have_form) break;
    if (nrun > 0 && (!have_form || dmin <= tf_next)) {
      // ---- COMPLETION (`simcore.py:173-198`)
      if (dmin < now - 1e-9) status |= INTF_ST_PAST_EVENT;
      now = now > dmin ? now : dmin;
      double c_start = R.start[0], c_total = R.total[0], c_prog = R.progress[0], c_tb = R.tb[0], c_sd = R.sd[0];
      int c_nseg = R.nseg[0], c_non1 = R.non1[0];
#pragma unroll
      for (int k = 1; k < CAPM; k++) {
        if (ci == k) {
          c_start = R.start[k];
          c_total = R.total[k];
          c_prog = R.progress[k];
          c_tb = R.tb[k];
          c_sd = R.sd[k];
          c_nseg = R.nseg[k];
          c_non1 = R.non1[k];
        }
      }
      if (now == c_tb) {
        c_nseg -= 1;
        c_non1 -= c_sd != 1.0 ? 1 : 0;
      } else {
        c_prog = c_prog + (now - c_tb) / c_sd;
      }
      if (fabs(c_prog - c_total) > 1e-6 * c_total) status |= INTF_ST_PROGRESS;
      const double measured = c_non1 == 0 ? c_total : now - c_start;  // `:181-185`
      actm &= ~(1u << ci);
      nrun--;
      // _colo_changed(survivors) (`simcore.py:143-146`): the chain continues here ...
#pragma unroll
      for (int k = 0; k < CAPM; k++) {
        if ((actm >> k) & 1u) {
          close(k);
          reseat(k);
        }
      }
      n_reseats += nrun;
      // ... while the completed batch's outputs are written (off the chain)
      B.b_start[ro + bmin] = c_start;
      B.b_completion[ro + bmin] = now;
      B.b_measured[ro + bmin] = measured;
      int nseg_c = c_nseg < B.seg_stride ? c_nseg : B.seg_stride;
      if (seg_cursor + nseg_c > J.seg_cap) {
        status |= INTF_ST_OVERFLOW;
        nseg_c = 0;
      }
      const int off = J.seg_base + seg_cursor;
      B.b_seg_off[ro + bmin] = off;
      B.b_nseg[ro + bmin] = nseg_c;
      for (int k = 0; k < nseg_c; k++) {
        const double* p = rec(ci, k);
        B.s_tbegin[off + k] = p[0];
        B.s_tend[off + k] = (k + 1 < nseg_c) ? rec(ci, k + 1)[0] : now;
        B.s_slowdown[off + k] = p[1];
        B.s_colo[3 * (size_t)(off + k) + 0] = p[2];
        B.s_colo[3 * (size_t)(off + k) + 1] = p[3];
        B.s_colo[3 * (size_t)(off + k) + 2] = p[4];
      }
      seg_cursor += nseg_c;
      // outcome order (completion, batch_id) (`simcore.py:305`)
      if (now != last_done) {
        B.out_order[ro + n_done] = bmin;
      } else {
        int pos = n_done;
        while (pos > J.b_lo) {
          const int prev = B.out_order[ro + pos - 1];
          if (B.b_completion[ro + prev] == now && prev > bmin) {
            B.out_order[ro + pos] = prev;
            pos--;
          } else {
            break;
          }
        }
        B.out_order[ro + pos] = bmin;
      }
      n_done++;
      last_done = now;
    } else {
      // ---- FORMATION: batch n_formed joins the FIFO dispatch queue
      now = now > tf_next ? now : tf_next;
      n_formed++;
      tf_next = n_formed < nb ? B.b_formed[ro + n_formed] : INFINITY;
    }
    // ---- try_dispatch (`simcore.py:258-262`) -> dispatch (`:153-171`)
    while (dq < n_formed && nrun < cap) {
      const int h = __ffs(~actm) - 1;  // a free slot (segment history region h)
#pragma unroll
      for (int k = 0; k < CAPM; k++) {
        if (k == h) {
          R.start[k] = now;
          R.total[k] = nx.total;
          R.progress[k] = 0.0;
          R.own0[k] = nx.own0;
          R.own1[k] = nx.own1;
          R.own2[k] = nx.own2;
#pragma unroll
          for (int q = 0; q < kScalarNz; q++) R.nz[k][q] = nx.nz[q];
          R.batch[k] = nx.b;
          R.nseg[k] = 0;
          R.non1[k] = 0;
          R.seq[k] = seqc;
        }
      }
      seqc++;
      const unsigned surv = actm;
      actm |= 1u << h;
      nrun++;
      if (B.b_running) B.b_running[ro + dq] = nrun;  // dispatch trace
      dq++;
      fetch_next(dq, nx);  // prefetch: consumed at the next dispatch
      // the new batch and the survivors (independent reseats)
#pragma unroll
      for (int k = 0; k < CAPM; k++) {
        if (k == h) {
          reseat(k);
        } else if ((surv >> k) & 1u) {
          close(k);
          reseat(k);
        }
      }
      n_reseats += nrun;
    }
  }
  if (nrun || dq < n_formed) status |= INTF_ST_NONQUIESCENT;
  ReplayJobOut r;
  r.status = status;
  r.n_segments = seg_cursor;
  r.n_reseats = n_reseats;
  r.last_done = last_done;
  return r;
}

}  // namespace intf
