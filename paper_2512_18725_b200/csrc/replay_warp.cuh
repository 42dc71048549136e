// replay_warp.cuh -- lane-group forms of the replay recurrence and of batch
// formation (sm_100a).  Same events, same arithmetic, same outputs as
// replay_formed() / form_scenario() in replay_core.cuh (which remain the
// readable, host-checkable statements).
//
// A replay job is mapped to a group of W lanes (W = 32 in use; W = 8 packs
// four jobs per warp), every collective is masked to the group:
//   * replay: lane l < cap owns running slot l in registers; the running
//     (dispatch) order is a group-uniform list of 4-bit lane ids, so each lane
//     computes its colo sum ((0 + p1) + p2).. in list order from shuffles and
//     all reseats of one event run in parallel (they are independent: colo
//     reads only `own`, noise is keyed by (batch, segment index)); the next
//     completion is a (done_at, batch_id) min over the cap lanes, compared
//     with the next formation as the reference heap would (completion first
//     at equal time);
//   * formation times, and the model/size/first noise draws of the batches
//     about to be dispatched, stream through W-batch register windows
//     refilled by coalesced loads, keeping global latency off the chain;
//   * formation: a warp per deployed model walks its arrival list (window
//     membership by ballot); a rank-merge on the heap key (time, kind, key)
//     assigns the scenario's global batch ids.
#pragma once
#include "replay_core.cuh"

namespace intf {

constexpr int kWarpNoiseK = 4;  // noise draws prefetched per dispatched batch
constexpr int kSmemSeg = 8;     // open-segment history kept in shared memory per slot (rest in global scratch)

// rare path (segment index beyond the precomputed noise table): kept out of
// line so the SeedSequence/PCG64 state does not inflate the replay's registers
__device__ __noinline__ double noise_draw_slow(uint64_t seed, uint64_t batch, uint64_t seg, double sigma) {
  return noise_draw(seed, batch, seg, sigma);
}

// W-lane group of the calling thread (W divides 32)
template <int W>
struct LaneGroup {
  unsigned mask;
  int lane, base;
  __device__ __forceinline__ LaneGroup() {
    const int l = threadIdx.x & 31;
    base = l & ~(W - 1);
    lane = l & (W - 1);
    mask = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << base);
  }
  __device__ __forceinline__ double shfl(double v, int src) const { return __shfl_sync(mask, v, src, W); }
  __device__ __forceinline__ int shfl(int v, int src) const { return __shfl_sync(mask, v, src, W); }
  __device__ __forceinline__ unsigned shfl(unsigned v, int src) const { return __shfl_sync(mask, v, src, W); }
  __device__ __forceinline__ double shfl_xor(double v, int o) const { return __shfl_xor_sync(mask, v, o, W); }
  __device__ __forceinline__ double shfl_up(double v, int d) const { return __shfl_up_sync(mask, v, d, W); }
  __device__ __forceinline__ int shfl_xor(int v, int o) const { return __shfl_xor_sync(mask, v, o, W); }
  __device__ __forceinline__ unsigned shfl_xor(unsigned v, int o) const { return __shfl_xor_sync(mask, v, o, W); }
  __device__ __forceinline__ unsigned ballot(bool p) const {
    const unsigned b = __ballot_sync(mask, p) >> base;
    return W == 32 ? b : (b & ((1u << W) - 1u));
  }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  __device__ __forceinline__ unsigned reduce_or(unsigned v) const { return __reduce_or_sync(mask, v); }
};

// One replay job: batches [b_lo, b_hi) of scenario s, started from an idle
// GPU, writing segments into [seg_base, seg_base + seg_cap) and using scratch
// slot `scratch`.  The whole-scenario replay is the job [0, n_batches).
struct ReplayJob {
  int s, b_lo, b_hi, seg_base, seg_cap, scratch;
};
struct ReplayJobOut {
  int status, n_segments, n_reseats;
  double last_done;
};

// ---------------------------------------------------------------------------
// concurrency_cap == 1: the same recurrence with nothing to co-locate.  Every
// batch runs alone, in FIFO (= batch id) order, as one segment [start, done)
// with colo = 0 and noise draw (b, 0):
//   start_b = max(now, formed_b)      (formation / completion event order, `simcore.py:246-262`)
//   done_b  = start_b + total_b * sd_b  (`_reseat` `simcore.py:141`, progress 0)
// so the serial chain per batch is one max and one add; the slowdowns, the
// products total*sd and every output are computed 32 batches at a time in
// parallel.  Same values, same rounding, same status checks as replay_group
// (zero-length pop, progress check, measured = total if sd == 1.0).
template <int W>
__device__ __noinline__ ReplayJobOut replay_cap1(const ReplayJob J, const intf_scenario& S,
                                                 const intf_model* __restrict__ md, const intf_table tab,
                                                 const intf_replay_buffers B, int status) {
  const LaneGroup<W> G;
  const int lane = G.lane;
  const int nb = J.b_hi, ro = S.req_off;
  double now = 0.0, last_done = -INFINITY;
  int seg_cursor = 0, n_reseats = 0;
  for (int base = J.b_lo; base < nb; base += W) {
    const int b = base + lane;
    const bool valid = b < nb;
    double tf = 0.0, w = 0.0, total = 1.0, sd = 1.0;
    if (valid) {
      const int entry = md[B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1;
      tf = B.b_formed[ro + b];
      total = tab.solo_ms[entry];
      const double own[3] = {tab.thr[3 * entry], tab.thr[3 * entry + 1], tab.thr[3 * entry + 2]};
      const double colo[3] = {0.0, 0.0, 0.0};
      const double noise = B.noise_k > 0 ? B.noise_tab[(size_t)(ro + b) * B.noise_k]
                                         : noise_draw_slow(S.oracle_seed, S.batch_id_base + (uint64_t)b, 0ull, S.sigma);
      sd = slowdown(own, colo, S.beta, noise);
      w = total * sd;  // remaining_work_ms * slowdown, remaining = total - 0.0
    }
    // the serial chain, uniform over the group (shuffles are off the chain)
    const int n = nb - base < W ? nb - base : W;
    double my_start = 0.0, my_done = 0.0;
#pragma unroll 8
    for (int i = 0; i < n; i++) {
      const double tfi = G.shfl(tf, i), wi = G.shfl(w, i);
      now = now > tfi ? now : tfi;  // formation (or the completion that freed the GPU)
      const double st = now;
      now = now + wi;               // completion: now = done
      if (i == lane) {
        my_start = st;
        my_done = now;
      }
    }
    // close_segment + complete (`simcore.py:56-66,173-198`), in parallel
    const bool kept = valid && my_done != my_start;  // zero-length segment is popped
    const double progress = kept ? 0.0 + (my_done - my_start) / sd : 0.0;
    if (valid && fabs(progress - total) > 1e-6 * total) status |= INTF_ST_PROGRESS;
    const double measured = (kept && sd != 1.0) ? my_done - my_start : total;
    const unsigned kmask = G.ballot(kept);
    const int before = __popc(kmask & ((1u << lane) - 1u));
    const int nkeep = __popc(kmask);
    const bool fits = seg_cursor + nkeep <= J.seg_cap;
    if (!fits) status |= INTF_ST_OVERFLOW;
    if (valid) {
      const int off = J.seg_base + seg_cursor + before;
      B.b_start[ro + b] = my_start;
      B.b_completion[ro + b] = my_done;
      B.b_measured[ro + b] = measured;
      B.b_seg_off[ro + b] = fits ? off : J.seg_base + seg_cursor;
      B.b_nseg[ro + b] = (kept && fits) ? 1 : 0;
      B.out_order[ro + b] = b;  // completions are non-decreasing in batch id
      if (B.b_running) B.b_running[ro + b] = 1;
      if (kept && fits) {
        B.s_tbegin[off] = my_start;
        B.s_tend[off] = my_done;
        B.s_slowdown[off] = sd;
        B.s_colo[3 * (size_t)off + 0] = 0.0;
        B.s_colo[3 * (size_t)off + 1] = 0.0;
        B.s_colo[3 * (size_t)off + 2] = 0.0;
      }
    }
    if (fits) seg_cursor += nkeep;
    n_reseats += n;
    last_done = now;
  }
  ReplayJobOut r;
  r.status = (int)G.reduce_or((unsigned)status);
  r.n_segments = seg_cursor;
  r.n_reseats = n_reseats;
  r.last_done = last_done;
  return r;
}

// sseg: this group's shared-memory segment history, [kMaxCap][kSmemSeg][5]
// CAPT > 0: the concurrency cap as a compile-time constant (unrolled
// running-list loops, constant reduction span); 0: runtime cap.
template <int W, int CAPT>
__device__ __forceinline__ ReplayJobOut replay_group_t(const ReplayJob J, const intf_scenario* __restrict__ scens,
                                                    const intf_model* __restrict__ models, const intf_table tab,
                                                    const intf_replay_buffers B, double* sseg, int status) {
  constexpr int KU = CAPT > 0 ? CAPT : kMaxCap;  // bound of the running-list loops
  const LaneGroup<W> G;
  const int lane = G.lane;
  const int s = J.s;
  const intf_scenario& S = scens[s];
  const int cap = CAPT > 0 ? CAPT : S.cap, nb = J.b_hi, ro = S.req_off;
  const intf_model* md = models + S.model_off;
  const int K = B.noise_k < kWarpNoiseK ? B.noise_k : kWarpNoiseK;
  double* myseg = B.slot_seg + ((size_t)J.scratch * B.cap_max + lane) * (size_t)B.seg_stride * 5;

  // ---- per-lane slot state (valid while `act`)
  bool act = false;
  double start = 0.0, total = 0.0, progress = 0.0, done = 0.0, own0 = 0.0, own1 = 0.0, own2 = 0.0;
  double cur_tb = 0.0, cur_sd = 1.0, cur_rsd = 1.0, nz0 = 1.0, nz1 = 1.0, nz2 = 1.0, nz3 = 1.0;
  int batch = 0, nseg = 0, n_non1 = 0;

  // ---- group-uniform state
  unsigned long long runlist = 0ull;  // 4-bit lane ids in dispatch order
  // (CAPT > 0) throughputs of the running batches, held by every lane: colo
  // sums without shuffles.  Cap 4: in running-list order.  Caps 2-3: by slot
  // (lane), because a batch has at most two peers there and the sum does not
  // depend on their order: ((0 + a) + b) == ((0 + b) + a) bit for bit (fp
  // addition commutes; 0 + x only maps -0 to +0), so the list order needs no
  // upkeep (no shifts at a completion, no list decode per reseat).
  constexpr bool kBySlot = CAPT == 2 || CAPT == 3;
  double u0[KU], u1[KU], u2[KU];
#pragma unroll
  for (int k = 0; k < KU; k++) u0[k] = u1[k] = u2[k] = 0.0;
  int nrun = 0;
  unsigned freemask = (cap >= 32) ? 0xffffffffu : ((1u << cap) - 1u);
  double now = 0.0;
  int n_formed = J.b_lo, dq = J.b_lo, n_done = J.b_lo, seg_cursor = 0, n_reseats = 0;
  double last_done = -INFINITY;  // completion time of the latest outcome
  bool refill = false;           // the completion just processed is followed by a dispatch

  // formation-time window: lane l holds b_formed of batch fbase + l
  int fbase = J.b_lo;
  double wf = fbase + lane < nb ? B.b_formed[ro + fbase + lane] : 0.0;
  // dispatch window: lane l holds the profile entry (solo ms, throughputs) and
  // the first noise draws of batch dbase + l, so a dispatch reads them by
  // shuffles instead of the dependent model -> entry -> table loads
  int dbase = J.b_lo;
  double wsol = 1.0, wt0 = 0.0, wt1 = 0.0, wt2 = 0.0;
  double wn0 = 1.0, wn1 = 1.0, wn2 = 1.0, wn3 = 1.0;
  auto load_dispatch_window = [&](int base) {
    const int b = base + lane;
    if (b < nb) {
      const int e = md[B.b_model[ro + b]].entry_base + B.b_size[ro + b] - 1;
      wsol = tab.solo_ms[e];
      wt0 = tab.thr[3 * e];
      wt1 = tab.thr[3 * e + 1];
      wt2 = tab.thr[3 * e + 2];
      const double* nt = B.noise_tab + (size_t)(ro + b) * B.noise_k;
      wn0 = K > 0 ? nt[0] : 1.0;
      wn1 = K > 1 ? nt[1] : 1.0;
      wn2 = K > 2 ? nt[2] : 1.0;
      wn3 = K > 3 ? nt[3] : 1.0;
    }
  };
  load_dispatch_window(J.b_lo);

  // reseat of this lane's batch at `now` (`simcore.py:133-141`); every lane of
  // the group calls it together (group-uniform shuffles inside)
  auto reseat_lane = [&](bool doit) {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    if constexpr (kBySlot) {
#pragma unroll
      for (int k = 0; k < KU; k++) {  // running peers by slot, skipping this lane's own batch
        if (k != lane && !((freemask >> k) & 1u)) {
          c0 = c0 + u0[k];
          c1 = c1 + u1[k];
          c2 = c2 + u2[k];
        }
      }
    } else if constexpr (CAPT > 0) {
#pragma unroll
      for (int k = 0; k < KU; k++) {  // running-list order, skipping this lane's own batch
        if (k < nrun && (int)((runlist >> (4 * k)) & 15ull) != lane) {
          c0 = c0 + u0[k];
          c1 = c1 + u1[k];
          c2 = c2 + u2[k];
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < KU; k++) {  // group-uniform loop, running-list order
        if (k >= nrun) break;
        const int j = (int)((runlist >> (4 * k)) & 15ull);
        const double a0 = G.shfl(own0, j), a1 = G.shfl(own1, j), a2 = G.shfl(own2, j);
        if (j != lane) {
          c0 = c0 + a0;
          c1 = c1 + a1;
          c2 = c2 + a2;
        }
      }
    }
    if (!doit) return;
    double noise;
    if (nseg < K) noise = nseg == 0 ? nz0 : nseg == 1 ? nz1 : nseg == 2 ? nz2 : nz3;
    else if (nseg < B.noise_k) noise = B.noise_tab[(size_t)(ro + batch) * B.noise_k + nseg];  // precomputed, L2
    else noise = noise_draw_slow(S.oracle_seed, S.batch_id_base + (uint64_t)batch, (uint64_t)nseg, S.sigma);
    const double o[3] = {own0, own1, own2}, colo[3] = {c0, c1, c2};
    const double sd = slowdown(o, colo, S.beta, noise);
    if (nseg < B.seg_stride) {
      double* p = nseg < kSmemSeg ? sseg + (lane * kSmemSeg + nseg) * 5 : myseg + (size_t)nseg * 5;
      p[0] = now;
      p[1] = sd;
      p[2] = c0;
      p[3] = c1;
      p[4] = c2;
    } else {
      status |= INTF_ST_SEG_STRIDE;
    }
    nseg++;
    cur_tb = now;
    cur_sd = sd;
    cur_rsd = 1.0 / sd;  // RN(1/sd), off the chain: the segment's close divides by sd
    if (sd != 1.0) n_non1++;
    done = now + (total - progress) * sd;
    if (done < now - 1e-9) status |= INTF_ST_PAST_EVENT;
  };
  // RunningBatch.close_segment (`simcore.py:56-66`)
  auto close_lane = [&]() {
    if (now == cur_tb) {
      nseg--;
      if (cur_sd != 1.0) n_non1--;
    } else {
      // (now - cur_tb) / cur_sd, correctly rounded (Markstein: with r = RN(1/y)
      // and q0 = RN(x r) within an ulp, RN(q0 + RN(x - y q0) r) = RN(x / y);
      // no overflow / underflow at these magnitudes): three dependent
      // multiply-adds on the chain instead of the division sequence
      const double x = now - cur_tb, q0 = x * cur_rsd;
      progress = progress + fma(fma(-cur_sd, q0, x), cur_rsd, q0);
    }
  };

  // butterfly span: slots live in lanes [0, cap), so log2(cap) rounds suffice
  int red_hi = 1;
  while (red_hi < cap) red_hi <<= 1;
  red_hi >>= 1;
  // next completion (CAPT > 0): kept across iterations that do not change the
  // running set (formations while the GPU is full)
  double dmin = INFINITY;
  int bmin = 0x7fffffff, cl_min = 0;
  bool min_ok = false;
  for (;;) {
    // next completion: lexicographic min of (done, batch) over active lanes
    if constexpr (CAPT > 0) {
      // slots live in lanes [0, CAPT): every lane reads all of them at once
      // (independent shuffles) and takes the min locally, with its lane
      if (!min_ok) {
        const double dv = act ? done : INFINITY;
        const int bv = act ? batch : 0x7fffffff;
        double dk[CAPT];
        int bk[CAPT];
#pragma unroll
        for (int k = 0; k < CAPT; k++) {
          dk[k] = G.shfl(dv, k);
          bk[k] = G.shfl(bv, k);
        }
        dmin = dk[0];
        bmin = bk[0];
        cl_min = 0;
#pragma unroll
        for (int k = 1; k < CAPT; k++) {
          if (dk[k] < dmin || (dk[k] == dmin && bk[k] < bmin)) {
            dmin = dk[k];
            bmin = bk[k];
            cl_min = k;
          }
        }
        min_ok = true;
      }
    } else {
      dmin = act ? done : INFINITY;
      bmin = act ? batch : 0x7fffffff;
      for (int o = red_hi; o > 0; o >>= 1) {
        const double d2 = G.shfl_xor(dmin, o);
        const int b2 = G.shfl_xor(bmin, o);
        if (d2 < dmin || (d2 == dmin && b2 < bmin)) {
          dmin = d2;
          bmin = b2;
        }
      }
      dmin = G.shfl(dmin, 0);
      bmin = G.shfl(bmin, 0);
    }
    const bool have_form = n_formed < nb;
    if (have_form && n_formed - fbase >= W) {
      fbase += W;
      wf = fbase + lane < nb ? B.b_formed[ro + fbase + lane] : 0.0;
    }
    const double tf = G.shfl(wf, (n_formed - fbase) & (W - 1));
    if (nrun == 0 && !have_form) break;
    if (nrun > 0 && (!have_form || dmin <= tf)) {
      // ---- COMPLETION (`simcore.py:173-198`)
      if (dmin < now - 1e-9) status |= INTF_ST_PAST_EVENT;
      now = now > dmin ? now : dmin;
      int cl;
      if constexpr (CAPT > 0) {
        cl = cl_min;
      } else {
        const unsigned cmask = G.ballot(act && batch == bmin);
        cl = __ffs(cmask) - 1;
      }
      min_ok = false;
      int nseg_c = 0, off = 0;
      // RunningBatch.close_segment of the completing batch (`simcore.py:174`)
      // and of every survivor (`:145`): independent, so one parallel step
      if (act) close_lane();
      if (lane == cl) {
        if (fabs(progress - total) > 1e-6 * total) status |= INTF_ST_PROGRESS;
        const double measured = n_non1 == 0 ? total : now - start;  // `:181-185`
        B.b_start[ro + batch] = start;
        B.b_completion[ro + batch] = now;
        B.b_measured[ro + batch] = measured;
        nseg_c = nseg < B.seg_stride ? nseg : B.seg_stride;
        if (seg_cursor + nseg_c > J.seg_cap) {
          status |= INTF_ST_OVERFLOW;
          nseg_c = 0;
        }
        off = J.seg_base + seg_cursor;
        B.b_seg_off[ro + batch] = off;
        B.b_nseg[ro + batch] = nseg_c;
        act = false;
      }
      G.sync();  // lane cl's outcome/segment writes visible to the group
      nseg_c = G.shfl(nseg_c, cl);
      off = G.shfl(off, cl);
      // lanes copy the completed batch's segments (segment k <- lane k mod W)
      const double* cseg = B.slot_seg + ((size_t)J.scratch * B.cap_max + cl) * (size_t)B.seg_stride * 5;
      const double* csm = sseg + cl * kSmemSeg * 5;
      for (int k = lane; k < nseg_c; k += W) {
        // every load before the first store (the history cannot alias the
        // outputs, but the compiler cannot know: interleaved, each store
        // would wait for its load on the chain); shared-memory rows by
        // shared-memory loads
        double v0, v1, v2, v3, v4, ve;
        if (k + 1 < kSmemSeg) {
          const double* p = csm + k * 5;
          v0 = p[0];
          v1 = p[1];
          v2 = p[2];
          v3 = p[3];
          v4 = p[4];
          ve = p[5];  // next row's t_begin
        } else {
          const double* p = k < kSmemSeg ? csm + k * 5 : cseg + (size_t)k * 5;
          const double* q = cseg + (size_t)(k + 1) * 5;
          v0 = p[0];
          v1 = p[1];
          v2 = p[2];
          v3 = p[3];
          v4 = p[4];
          ve = k + 1 < nseg_c ? q[0] : now;
        }
        if (k + 1 >= nseg_c) ve = now;
        B.s_tbegin[off + k] = v0;
        B.s_tend[off + k] = ve;
        B.s_slowdown[off + k] = v1;
        B.s_colo[3 * (size_t)(off + k) + 0] = v2;
        B.s_colo[3 * (size_t)(off + k) + 1] = v3;
        B.s_colo[3 * (size_t)(off + k) + 2] = v4;
      }
      seg_cursor += nseg_c;
      // outcome order (completion, batch_id) (`simcore.py:305`): only runs of
      // equal completion time can need an insertion
      if (lane == 0 && now != last_done) {
        B.out_order[ro + n_done] = bmin;  // strictly later than every earlier outcome
      } else if (lane == 0) {
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
      G.sync();
      n_done++;
      last_done = now;
      // remove cl from the running list, keep order
      if constexpr (kBySlot) {
        nrun--;
      } else {
        unsigned long long nl = 0ull;
        int w = 0, pc = 0;
#pragma unroll
        for (int k = 0; k < KU; k++) {
          if (k >= nrun) break;
          const unsigned long long j = (runlist >> (4 * k)) & 15ull;
          if ((int)j != cl) nl |= j << (4 * w++);
          else pc = k;
        }
        runlist = nl;
        nrun = w;
        if constexpr (CAPT > 0) {
#pragma unroll
        for (int k = 0; k + 1 < KU; k++) {
          if (k >= pc) {
            u0[k] = u0[k + 1];
            u1[k] = u1[k + 1];
            u2[k] = u2[k + 1];
          }
        }
        }
      }
      freemask |= 1u << cl;
      // _colo_changed(survivors) (`simcore.py:143-146`): closed above;
      // a queued batch dispatches at this same instant and reseats every
      // survivor again; the reseat here would open a zero-length segment that
      // the dispatch pops (same noise index, progress and counts restored), so
      // only the dispatch's reseat is computed (both are counted)
      refill = dq < n_formed;
      if (!refill) reseat_lane(act);
      n_reseats += nrun;
    } else if (nrun == cap) {
      // ---- FORMATIONS while the GPU is full: until the next completion they
      // only lengthen the FIFO queue (try_dispatch cannot dispatch), so every
      // formation before dmin (strictly: a completion at the same instant
      // goes first) is consumed at once, now = max(now, its time)
      for (;;) {
        const int off = n_formed - fbase;  // window lane of the next formation
        // formation times are non-decreasing: the qualifying lanes are contiguous from `off`
        const unsigned q = G.ballot(lane >= off && fbase + lane < nb && wf < dmin);
        const int cnt = __popc(q);
        if (cnt == 0) break;
        const double tl = G.shfl(wf, off + cnt - 1);
        now = now > tl ? now : tl;
        n_formed += cnt;
        if (n_formed >= nb || off + cnt < W) break;  // stopped inside this window
        fbase += W;
        wf = fbase + lane < nb ? B.b_formed[ro + fbase + lane] : 0.0;
      }
    } else {
      // ---- FORMATION: batch n_formed joins the FIFO dispatch queue
      now = now > tf ? now : tf;
      n_formed++;
    }
    // ---- try_dispatch (`simcore.py:258-262`) -> dispatch (`:153-171`)
    while (dq < n_formed && nrun < cap) {
      const int b = dq++;
      if (b - dbase >= W) {
        dbase += W;
        load_dispatch_window(dbase);
      }
      const int src = (b - dbase) & (W - 1);
      const double t0 = G.shfl(wt0, src), t1 = G.shfl(wt1, src), t2 = G.shfl(wt2, src), sol = G.shfl(wsol, src);
      const double n0 = G.shfl(wn0, src), n1 = G.shfl(wn1, src), n2 = G.shfl(wn2, src), n3 = G.shfl(wn3, src);
      min_ok = false;
      const int L = __ffs(freemask) - 1;
      freemask &= ~(1u << L);
      if constexpr (!kBySlot) runlist |= (unsigned long long)L << (4 * nrun);
      nrun++;
      const bool was_act = act;
      if constexpr (CAPT > 0) {  // every lane records the new batch's throughputs
#pragma unroll
        for (int k = 0; k < KU; k++) {
          if (k == (kBySlot ? L : nrun - 1)) {
            u0[k] = t0;
            u1[k] = t1;
            u2[k] = t2;
          }
        }
      }
      if (lane == L) {
        if (B.b_running) B.b_running[ro + b] = nrun;  // dispatch trace
        act = true;
        batch = b;
        start = now;
        total = sol;
        progress = 0.0;
        nseg = 0;
        n_non1 = 0;
        own0 = t0;
        own1 = t1;
        own2 = t2;
        nz0 = n0;
        nz1 = n1;
        nz2 = n2;
        nz3 = n3;
      }
      // new batch first, then survivors: independent, so in parallel
      if (was_act && !refill) close_lane();  // (after a completion that refills: already closed)
      refill = false;
      reseat_lane(act);
      n_reseats += nrun;
    }
  }
  if (nrun || dq < n_formed) status |= INTF_ST_NONQUIESCENT;
  ReplayJobOut r;
  r.status = (int)G.reduce_or((unsigned)status);
  r.n_segments = seg_cursor;
  r.n_reseats = n_reseats;
  r.last_done = last_done;
  return r;
}

// the replay of one job: dispatch on the concurrency cap (uniform per group)
template <int W>
__device__ __forceinline__ ReplayJobOut replay_group(const ReplayJob J, const intf_scenario* __restrict__ scens,
                                                     const intf_model* __restrict__ models, const intf_table tab,
                                                     const intf_replay_buffers B, double* sseg, int status) {
  const intf_scenario& S = scens[J.s];
  switch (S.cap) {
    case 1: return replay_cap1<W>(J, S, models + S.model_off, tab, B, status);
    case 2: return replay_group_t<W, 2>(J, scens, models, tab, B, sseg, status);
    case 3: return replay_group_t<W, 3>(J, scens, models, tab, B, sseg, status);
    case 4: return replay_group_t<W, 4>(J, scens, models, tab, B, sseg, status);
    default: return replay_group_t<W, 0>(J, scens, models, tab, B, sseg, status);
  }
}

// ---------------------------------------------------------------------------
// A model's next formation event from list index h, computed by a lane group:
// the window membership test t < D is monotone along the sorted list, so the
// member count is a ballot popcount (same result as next_formation()).
template <int W>
__device__ __forceinline__ void group_next_formation(const LaneGroup<W>& G, const double* lt, const int32_t* lrid,
                                                     int n, int h, double window, int max_bs, uint32_t crc,
                                                     double& t, int& kind, uint32_t& key, int& cnt) {
  if (h >= n) {
    kind = 0;
    t = 0.0;
    key = 0;
    cnt = 0;
    return;
  }
  const double D = lt[h] + window;  // every lane loads the same word (broadcast)
  int c = 1;
  for (int j0 = 1; j0 < max_bs; j0 += W) {
    const int j = j0 + G.lane;
    const bool in = j < max_bs && h + j < n && lt[h + j] < D;
    const int add = __popc(G.ballot(in));
    c += add;
    if (add < W) break;
  }
  cnt = c;
  if (c == max_bs) {
    t = lt[h + c - 1];
    kind = KIND_ARRIVAL;
    key = (uint32_t)lrid[h + c - 1];
  } else {
    t = D;
    kind = KIND_WINDOW;
    key = crc;
  }
}

// ---------------------------------------------------------------------------
// Per-model formation (warp per deployed model): a model's batch sequence
// depends only on its own arrivals and window, so every
// model forms its batches in parallel into per-model lists of
// (time, kind, key) + (count, head).  A rank-merge then orders all batches
// of a scenario exactly as the reference heap pops formation events.
// One model's batches by a W-lane group, max_batch_size <= W: the arrival
// list streams through a 2W-element register window (two coalesced loads per
// W heads), the head time and the members come from shuffles and ballots (no
// global load on the h -> h + cnt chain), and the events are held one per
// lane and flushed W at a time with coalesced stores.  next_formation's rule:
// cnt = 1 + #(t[h+j] < t[h] + window), 0 < j < max_bs (sorted: a prefix).
template <int W>
__device__ __forceinline__ void form_model_win(const LaneGroup<W>& G, const intf_scenario& S, const intf_model& Md,
                                               int n_list, const intf_replay_buffers& B, int g) {
  const double* lt = B.list_t + Md.list_off;
  const int32_t* lrid = B.list_rid + Md.list_off;
  const int lane = G.lane;
  int h = 0, c = 0, base = 0;
  double w0 = lane < n_list ? lt[lane] : INFINITY, w1 = W + lane < n_list ? lt[W + lane] : INFINITY;
  int r0 = lane < n_list ? lrid[lane] : 0, r1 = W + lane < n_list ? lrid[W + lane] : 0;  // request ids
  double ot = 0.0;
  int okind = 0, okey = 0, ocnt = 0, oh = 0;
  auto flush = [&](int c0, int k) {
    if (lane < k) {
      B.mb_t[Md.list_off + c0 + lane] = ot;
      reinterpret_cast<int4*>(B.mb_info)[Md.list_off + c0 + lane] = make_int4(okind, okey, ocnt, oh);
    }
  };
  while (h < n_list) {
    if (h - base >= W) {  // cnt <= max_bs <= W: one slide keeps h inside [base, base + W)
      base += W;
      w0 = w1;
      r0 = r1;
      w1 = base + W + lane < n_list ? lt[base + W + lane] : INFINITY;
      r1 = base + W + lane < n_list ? lrid[base + W + lane] : 0;
    }
    const int o = h - base;
    const double D = G.shfl(w0, o) + S.window_ms;  // arm_window at the first arrival (`batcher.py:66-68`)
    const int lim = min(o + S.max_bs, n_list - base);  // window offsets (o, lim) may join
    const unsigned m0 = G.ballot(lane > o && lane < lim && w0 < D);
    const unsigned m1 = G.ballot(W + lane > o && W + lane < lim && w1 < D);
    const int cnt = 1 + __popc(m0) + __popc(m1);
    const int last = o + cnt - 1;
    const double tl = last < W ? G.shfl(w0, last) : G.shfl(w1, last - W);
    const int rl = last < W ? G.shfl(r0, last) : G.shfl(r1, last - W);
    if (lane == (c & (W - 1))) {  // batch c's event, held by lane c % W
      if (cnt == S.max_bs) {  // early emit at max_batch_size (`batcher.py:70-71`)
        ot = tl;
        okind = KIND_ARRIVAL;
        okey = rl;
      } else {  // window expiry (`batcher.py:74-85`)
        ot = D;
        okind = KIND_WINDOW;
        okey = (int32_t)Md.crc;
      }
      ocnt = cnt;
      oh = h;
    }
    h += cnt;
    c++;
    if ((c & (W - 1)) == 0) flush(c - W, W);
  }
  if (c & (W - 1)) flush(c & ~(W - 1), c & (W - 1));
  if (lane == 0) B.n_mb[g] = c;
}

// The same batches with the per-head work taken off the chain: the warp loads
// the 64 arrivals from the current head h, and lane l computes the batch that
// WOULD start at head h + l -- its member count (1 + #(t[h+l+j] < t[h+l] +
// window), 0 < j < max_bs, a prefix of the sorted list), its event time, kind
// and key -- for all 32 candidate heads at once (max_bs - 1 shuffles).  The
// serial chain h -> h + cnt(h) then costs one shuffle per batch; the lanes
// on the chain are the batches, which write their events directly to their
// output slots (consecutive lanes -> consecutive slots).  Every iteration
// advances at least 32 arrivals.  Same recurrence as form_model_win.
__device__ __forceinline__ void form_model_heads(const intf_scenario& S, const intf_model& Md, int n_list,
                                                 const intf_replay_buffers& B, int g) {
  const double* lt = B.list_t + Md.list_off;
  const int32_t* lrid = B.list_rid + Md.list_off;
  const int lane = threadIdx.x & 31;
  const int mbs = S.max_bs;
  int h = 0, c = 0;
  while (h < n_list) {
    const double w0 = h + lane < n_list ? lt[h + lane] : INFINITY;
    const double w1 = h + 32 + lane < n_list ? lt[h + 32 + lane] : INFINITY;
    const int r0 = h + lane < n_list ? lrid[h + lane] : 0;
    const int r1 = h + 32 + lane < n_list ? lrid[h + 32 + lane] : 0;
    // the batch starting at head h + lane: 1 + the number of following
    // arrivals before its window closes, a prefix of the sorted list -- the
    // first j in [1, max_bs) with t[h + lane + j] >= D by binary search
    // (5 probes instead of max_bs - 1)
    const double D = w0 + S.window_ms;  // arm_window at the first arrival (`batcher.py:66-68`)
    int lo = 1, hi = mbs;
#pragma unroll
    for (int step = 0; step < 5; step++) {  // 2^5 >= max_bs - 1 (this form: max_bs <= 32)
      const int mid = (lo + hi) >> 1;
      const int src = lane + mid;  // window element lane + mid (< 64): w0 of lane src, or w1 of lane src - 32
      const double a = __shfl_sync(0xffffffffu, w0, src & 31), b = __shfl_sync(0xffffffffu, w1, src & 31);
      const double v = src < 32 ? a : b;
      if (lo < hi) {
        if (v < D) lo = mid + 1;
        else hi = mid;
      }
    }
    const int cnt = lo;
    const int last = lane + cnt - 1;  // < 64
    const double ta = __shfl_sync(0xffffffffu, w0, last & 31), tb = __shfl_sync(0xffffffffu, w1, last & 31);
    const int ra = __shfl_sync(0xffffffffu, r0, last & 31), rb = __shfl_sync(0xffffffffu, r1, last & 31);
    const bool full = cnt == mbs;  // early emit at max_batch_size (`batcher.py:70-71`), else window expiry
    const double et = full ? (last < 32 ? ta : tb) : D;
    const int ekind = full ? KIND_ARRIVAL : KIND_WINDOW;
    const int ekey = full ? (last < 32 ? ra : rb) : (int32_t)Md.crc;
    // walk the chain from offset 0 while the head lies in this window
    unsigned heads = 0u;
    int o = 0;
    while (o < 32 && h + o < n_list) {
      heads |= 1u << o;
      o += __shfl_sync(0xffffffffu, cnt, o);
    }
    if ((heads >> lane) & 1u) {
      const int idx = c + __popc(heads & ((1u << lane) - 1u));
      B.mb_t[Md.list_off + idx] = et;
      reinterpret_cast<int4*>(B.mb_info)[Md.list_off + idx] = make_int4(ekind, ekey, cnt, h + lane);
    }
    c += __popc(heads);
    h += o;
  }
  if (lane == 0) B.n_mb[g] = c;
}

// Per-model formation by a warp (max_batch_size > 32: the original walk with
// global loads; <= 32: the head-parallel form).  A rank-merge then orders all
// batches of a scenario exactly as the reference heap pops formation events.
__device__ __forceinline__ void form_model_warp(const intf_scenario& S, const intf_model& Md, int n_list,
                                                const intf_replay_buffers& B, int g) {
  const LaneGroup<32> G;
  if (S.max_bs <= 32) {
#ifdef INTF_FORM_WIN
    form_model_win<32>(G, S, Md, n_list, B, g);
#else
    form_model_heads(S, Md, n_list, B, g);
#endif
    return;
  }
  const double* lt = B.list_t + Md.list_off;
  const int32_t* lrid = B.list_rid + Md.list_off;
  int h = 0, c = 0;
  for (;;) {
    double t;
    int kind, cnt;
    uint32_t key;
    group_next_formation<32>(G, lt, lrid, n_list, h, S.window_ms, S.max_bs, Md.crc, t, kind, key, cnt);
    if (!kind) break;
    if (G.lane == 0) {
      B.mb_t[Md.list_off + c] = t;
      int32_t* info = B.mb_info + 4ll * (Md.list_off + c);
      info[0] = kind;
      info[1] = (int32_t)key;
      info[2] = cnt;
      info[3] = h;
    }
    h += cnt;
    c++;
  }
  if (G.lane == 0) B.n_mb[g] = c;
}

// lexicographic heap key of a formation event
__device__ __forceinline__ bool form_key_less(double t1, int k1, uint32_t y1, double t2, int k2, uint32_t y2) {
  return t1 < t2 || (t1 == t2 && (k1 < k2 || (k1 == k2 && y1 < y2)));
}

// number of batches in a per-model list that precede (t, kind, key)
__device__ __forceinline__ int count_form_before(const double* mt, const int32_t* mi, int n, double t, int kind,
                                                 uint32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (form_key_less(mt[mid], mi[4 * mid], (uint32_t)mi[4 * mid + 1], t, kind, key)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// Warp-cooperative arrival stream of one deployed model (`workload.py:80-94`).
// Lane l produces draws l, l+32, ... of the model's PCG64 stream using LCG
// jump-ahead (state_{i+1} = A_{i+1} state_0 + C_{i+1}; stride 32 with
// (A_32, C_32)), so the RNG and glibc log1p run 32-wide; the cumulative sum
// t += max(gap, 1e-12) stays strictly sequential (one lane, shared memory),
// exactly as the reference rounds it.
__device__ __forceinline__ void lcg_pow(unsigned __int128 mult, unsigned __int128 inc, unsigned long long n,
                                       unsigned __int128& A, unsigned __int128& C) {
  // (A, C) such that n steps of x -> mult*x + inc equal x -> A*x + C
  unsigned __int128 acc_mult = 1, acc_plus = 0, cur_mult = mult, cur_plus = inc;
  while (n) {
    if (n & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    n >>= 1;
  }
  A = acc_mult;
  C = acc_plus;
}

__device__ __forceinline__ uint64_t pcg_output(unsigned __int128 st) {
  const uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
  const uint32_t rot = (uint32_t)(hi >> 58);
  const uint64_t v = hi ^ lo;
  return (v >> rot) | (v << ((64u - rot) & 63u));
}

// returns the count; writes at most list_cap times; gaps: 32 doubles of smem
__device__ __noinline__ int gen_model_arrivals_warp(const intf_scenario& S, const intf_model& M, double* list_t,
                                                    int list_cap, volatile double* gaps) {
  const int lane = threadIdx.x & 31;
  if (M.rate_rps == 0.0) return 0;
  uint32_t w[4];
  int nw = push_words(w, 0, S.seed);
  nw = push_words(w, nw, M.crc);
  Pcg64 g = pcg_seed_words(w, nw);
  const unsigned __int128 mult =
      ((unsigned __int128)0x2360ed051fc65da4ull << 64) | (unsigned __int128)0x4385df649fccf645ull;
  unsigned __int128 Al, Cl, A32, C32;
  lcg_pow(mult, g.inc, (unsigned long long)(lane + 1), Al, Cl);
  lcg_pow(mult, g.inc, 32ull, A32, C32);
  unsigned __int128 st = Al * g.state + Cl;  // state after lane+1 steps
  const double horizon = S.duration_s * 1000.0;
  const double neg_mean_gap = -(1000.0 / M.rate_rps);
  double t = 0.0;  // running time (lane 0 keeps the authoritative copy)
  int n = 0;
  for (;;) {
    const double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
    st = A32 * st + C32;
    const double gap = neg_mean_gap * glibc_log1p(-u);
    gaps[lane] = gap > 1e-12 ? gap : 1e-12;
    __syncwarp();
    if (lane == 0) {
      double tt = t;
#pragma unroll 8
      for (int k = 0; k < 32; k++) {
        tt = tt + gaps[k];
        gaps[k] = tt;
      }
      t = tt;
    }
    __syncwarp();
    const double tl = gaps[lane];
    const unsigned inside = __ballot_sync(0xffffffffu, tl < horizon);
    // times are non-decreasing: the first t >= horizon ends the stream
    const int k_in = __popc(inside) == 32 ? 32 : __ffs(~inside) - 1;
    if (lane < k_in && n + lane < list_cap) list_t[n + lane] = tl;
    n += k_in;
    if (k_in < 32) break;
    t = __shfl_sync(0xffffffffu, t, 0);
    __syncwarp();
  }
  return n;
}

}  // namespace intf
