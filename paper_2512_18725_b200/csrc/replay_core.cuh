// replay_core.cuh -- per-scenario scheduler replay as a heap-free recurrence.
//
// Reference: `simcore.py:218-310` drives a binary heap of (time, kind, key,
// seq) events -- COMPLETION(0,batch_id) < WINDOW(1,crc32(model)) <
// ARRIVAL(2,request_id) -- with stale-event skipping, `batcher.py:44-85`
// queues and a FIFO dispatch queue.  Two facts let a GPU thread replace the
// heap by O(models + cap) state:
//   1. batch formation never reads GPU state, and every non-stale WINDOW
//      event forms a batch; so each model's next formation event is a pure
//      function of its arrival list and window: from head h,
//        D = t[h] + window;  members = h.. while t < D, at most max_bs;
//        full -> (t[last], ARRIVAL, request_id(last)), else (D, WINDOW, crc32);
//   2. dispatch order is batch-id (formation) order, and after every event
//      the dispatch queue is empty or the running set is full, so
//      try_dispatch only matters after completions and formations.
// The next event is therefore min over {<= cap live completions (done_at,
// batch_id)} U {<= n_models formation events}, compared as the heap would.
// Arrival/stale events that only advance `now` are dominated by the next
// real event's time (heap order), so skipping them is exact.
//
// Arithmetic is the reference's, operation for operation (-fmad=false):
//   colo    = ((0 + p1) + p2) + ...  in running-list order     `simcore.py:126-131`
//   slowdown= (1 + fma-chain(beta, max(0, own+colo-1))) * noise  `oracle.py:42-47`
//   done_at = now + (total - progress) * slowdown               `simcore.py:139-140`
//   close   : t == t_begin -> pop; else progress += (t-t_begin)/slowdown  `:56-66`
//   noise index = segment count after pops (index reuse)          `:135`
//   now = max(now, t)                                             `:207`
#pragma once
#include "../../include/intfsim_b200.h"
#include "intf_device.cuh"

namespace intf {

enum { KIND_COMPLETION = 0, KIND_WINDOW = 1, KIND_ARRIVAL = 2 };
constexpr int kMaxModels = 32;
constexpr int kMaxCap = 8;

// ---------------------------------------------------------------- arrivals
// generate_arrivals for ONE deployed model (`workload.py:80-94`): returns the
// count; writes at most list_cap times.
INTF_FN int gen_model_arrivals(const intf_scenario& S, const intf_model& M, double* list_t, int list_cap) {
  if (M.rate_rps == 0.0) return 0;
  uint32_t w[4];
  int nw = push_words(w, 0, S.seed);
  nw = push_words(w, nw, M.crc);
  Pcg64 g = pcg_seed_words(w, nw);
  const double horizon = S.duration_s * 1000.0;
  const double neg_mean_gap = -(1000.0 / M.rate_rps);
  double t = 0.0;
  int n = 0;
  for (;;) {
    double gap = neg_mean_gap * glibc_log1p(-pcg_next_double(g));
    t += gap > 1e-12 ? gap : 1e-12;
    if (t >= horizon) break;
    if (n < list_cap) list_t[n] = t;
    n++;
  }
  return n;
}

// number of elements of sorted list (t', rank') that precede (t, rank)
INTF_FN int count_before(const double* lt, int n, double t, bool ties_before) {
  int lo = 0, hi = n;  // first index with lt >= t (or > t if ties_before)
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    bool before = ties_before ? (lt[mid] <= t) : (lt[mid] < t);
    if (before) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ------------------------------------------------------------------ replay
struct FormEv {
  double t;
  uint32_t key;
  int32_t kind;  // 1 window, 2 arrival; 0 = none
  int32_t cnt;
};

INTF_FN bool form_less(const FormEv& a, const FormEv& b) {
  if (a.t != b.t) return a.t < b.t;
  if (a.kind != b.kind) return a.kind < b.kind;
  return a.key < b.key;
}

// next formation event of a model whose first unbatched list index is h
INTF_FN FormEv next_formation(const double* lt, const int32_t* lrid, int n, int h, double window, int max_bs,
                              uint32_t crc) {
  FormEv e;
  if (h >= n) {
    e.kind = 0;
    e.t = 0.0;
    e.key = 0;
    e.cnt = 0;
    return e;
  }
  const double D = lt[h] + window;  // arm_window at the first arrival (`batcher.py:66-68`)
  int cnt = 1;
  while (cnt < max_bs && h + cnt < n && lt[h + cnt] < D) cnt++;
  e.cnt = cnt;
  if (cnt == max_bs) {  // early emit at max_batch_size (`batcher.py:70-71`)
    e.t = lt[h + cnt - 1];
    e.kind = KIND_ARRIVAL;
    e.key = (uint32_t)lrid[h + cnt - 1];
  } else {  // window expiry (`batcher.py:74-85`)
    e.t = D;
    e.kind = KIND_WINDOW;
    e.key = crc;
  }
  return e;
}

struct Slot {
  double start, total, progress, done, own[3];
  double cur_tb, cur_sd;  // the open (last) segment, mirrored from scratch
  int32_t batch, entry, nseg, n_non1;
};

struct ReplayCtx {
  const intf_scenario* S;
  const intf_table* tab;
  const intf_replay_buffers* buf;
  double* seg;  // this scenario's slot scratch: [cap][seg_stride][5]
  int32_t status, n_reseats;
};

INTF_FN double* seg_ptr(ReplayCtx& c, int slot, int k) {
  return c.seg + ((size_t)slot * (size_t)c.buf->seg_stride + (size_t)k) * 5;
}

// GpuState._reseat (`simcore.py:133-141`)
INTF_FN void reseat(ReplayCtx& c, Slot* slots, const int* run, int nrun, int si, double now) {
  Slot& rb = slots[si];
  double colo[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < nrun; i++) {
    if (run[i] == si) continue;
    const Slot& o = slots[run[i]];
    colo[0] = colo[0] + o.own[0];
    colo[1] = colo[1] + o.own[1];
    colo[2] = colo[2] + o.own[2];
  }
  const intf_scenario& S = *c.S;
  double noise;
  if (rb.nseg < c.buf->noise_k)  // precomputed by k_noise_table (same draw)
    noise = c.buf->noise_tab[(size_t)(S.req_off + rb.batch) * c.buf->noise_k + rb.nseg];
  else
    noise = noise_draw(S.oracle_seed, S.batch_id_base + (uint64_t)rb.batch, (uint64_t)rb.nseg, S.sigma);
  double sd = slowdown(rb.own, colo, S.beta, noise);
  if (rb.nseg >= c.buf->seg_stride) {
    c.status |= INTF_ST_SEG_STRIDE;
  } else {
    double* p = seg_ptr(c, si, rb.nseg);
    p[0] = now;
    p[1] = sd;
    p[2] = colo[0];
    p[3] = colo[1];
    p[4] = colo[2];
  }
  rb.nseg++;
  rb.cur_tb = now;
  rb.cur_sd = sd;
  if (sd != 1.0) rb.n_non1++;
  c.n_reseats++;
  rb.done = now + (rb.total - rb.progress) * sd;
  if (rb.done < now - 1e-9) c.status |= INTF_ST_PAST_EVENT;
}

// RunningBatch.close_segment (`simcore.py:56-66`)
INTF_FN void close_segment(ReplayCtx& c, Slot& rb, int si, double now) {
  (void)c;
  (void)si;
  if (now == rb.cur_tb) {  // zero-length interval: drop it, reuse its index
    rb.nseg--;
    if (rb.cur_sd != 1.0) rb.n_non1--;
    return;
  }
  rb.progress = rb.progress + (now - rb.cur_tb) / rb.cur_sd;
}

// Batch formation for scenario s (`batcher.py:44-85` + the WINDOW/ARRIVAL
// branches of `simcore.py:246-256,289-299`): merges the per-model formation
// events in heap order (time, kind, key) and assigns global batch ids.
// Writes b_model, b_size, b_formed, r_batch and n_batches.  GPU-state free.
INTF_FN void form_scenario(int s, const intf_scenario* scens, const intf_model* models,
                           const intf_replay_buffers& B) {
  const intf_scenario& S = scens[s];
  const int M = S.n_models;
  if (M > kMaxModels || S.cap > B.cap_max || S.cap > kMaxCap || S.cap < 1 || S.max_bs < 1) {
    B.status[s] = INTF_ST_CAP;
    B.n_batches[s] = 0;
    return;
  }
  const intf_model* md = models + S.model_off;
  FormEv ev[kMaxModels];
  int head[kMaxModels];
  for (int m = 0; m < M; m++) {
    head[m] = 0;
    ev[m] = next_formation(B.list_t + md[m].list_off, B.list_rid + md[m].list_off, B.n_list[S.model_off + m], 0,
                           S.window_ms, S.max_bs, md[m].crc);
  }
  const int ro = S.req_off;
  int n_formed = 0;
  for (;;) {
    int fm = -1;
    for (int m = 0; m < M; m++)
      if (ev[m].kind && (fm < 0 || form_less(ev[m], ev[fm]))) fm = m;
    if (fm < 0) break;
    const FormEv e = ev[fm];
    const intf_model& mm = md[fm];
    const int b = n_formed++;
    B.b_model[ro + b] = fm;
    B.b_size[ro + b] = e.cnt;
    B.b_formed[ro + b] = e.t;
    const int32_t* lrid = B.list_rid + mm.list_off;
    for (int j = 0; j < e.cnt; j++) B.r_batch[ro + lrid[head[fm] + j]] = b;
    head[fm] += e.cnt;
    ev[fm] = next_formation(B.list_t + mm.list_off, lrid, B.n_list[S.model_off + fm], head[fm], S.window_ms,
                            S.max_bs, mm.crc);
  }
  B.n_batches[s] = n_formed;
}

// The replay proper for scenario s over its formed batches: FIFO capped
// admission, reseats, completions, outcome order.  Formation events are the
// batches in id order (their (time, kind, key) order was resolved by
// form_scenario); a completion precedes a formation at equal time (kind 0).
INTF_FN void replay_formed(int s, const intf_scenario* scens, const intf_model* models, const intf_table& tab,
                           const intf_replay_buffers& B) {
  const intf_scenario& S = scens[s];
  ReplayCtx c;
  c.S = &S;
  c.tab = &tab;
  c.buf = &B;
  c.seg = B.slot_seg + (size_t)s * (size_t)B.cap_max * (size_t)B.seg_stride * 5;
  c.status = B.status[s];
  c.n_reseats = 0;
  if (c.status & INTF_ST_CAP) return;
  const intf_model* md = models + S.model_off;
  const int nb = B.n_batches[s];
  Slot slots[kMaxCap];
  int run[kMaxCap], free_slots[kMaxCap], nfree = S.cap, nrun = 0;
  for (int i = 0; i < S.cap; i++) free_slots[i] = S.cap - 1 - i;
  double now = 0.0;
  int n_formed = 0, dq = 0, n_done = 0, seg_cursor = 0;
  const int ro = S.req_off;

  for (;;) {
    int ci = -1;
    for (int i = 0; i < nrun; i++) {
      if (ci < 0) {
        ci = i;
        continue;
      }
      const Slot& a = slots[run[i]];
      const Slot& b = slots[run[ci]];
      if (a.done < b.done || (a.done == b.done && a.batch < b.batch)) ci = i;
    }
    const bool have_form = n_formed < nb;
    if (ci < 0 && !have_form) break;
    if (ci >= 0 && (!have_form || slots[run[ci]].done <= B.b_formed[ro + n_formed])) {
      // ---- COMPLETION (`simcore.py:173-198`, `:283-288`)
      const int si = run[ci];
      Slot& rb = slots[si];
      if (rb.done < now - 1e-9) c.status |= INTF_ST_PAST_EVENT;
      now = now > rb.done ? now : rb.done;
      close_segment(c, rb, si, now);
      if (fabs(rb.progress - rb.total) > 1e-6 * rb.total) c.status |= INTF_ST_PROGRESS;
      for (int i = ci; i + 1 < nrun; i++) run[i] = run[i + 1];
      nrun--;
      free_slots[nfree++] = si;
      double measured = now - rb.start;
      if (rb.n_non1 == 0) measured = rb.total;  // all slowdowns == 1.0 (`:181-185`)
      const int b = rb.batch;
      B.b_start[ro + b] = rb.start;
      B.b_completion[ro + b] = now;
      B.b_measured[ro + b] = measured;
      const int nseg = rb.nseg < B.seg_stride ? rb.nseg : B.seg_stride;
      if (seg_cursor + nseg > S.seg_cap) {
        c.status |= INTF_ST_OVERFLOW;
        B.b_seg_off[ro + b] = S.seg_off;
        B.b_nseg[ro + b] = 0;
      } else {
        const int off = S.seg_off + seg_cursor;
        B.b_seg_off[ro + b] = off;
        B.b_nseg[ro + b] = nseg;
        for (int k = 0; k < nseg; k++) {
          const double* p = seg_ptr(c, si, k);
          B.s_tbegin[off + k] = p[0];
          B.s_tend[off + k] = (k + 1 < nseg) ? seg_ptr(c, si, k + 1)[0] : now;
          B.s_slowdown[off + k] = p[1];
          B.s_colo[3 * (off + k) + 0] = p[2];
          B.s_colo[3 * (off + k) + 1] = p[3];
          B.s_colo[3 * (off + k) + 2] = p[4];
        }
        seg_cursor += nseg;
      }
      // outcome order: sort key (completion, batch_id) (`simcore.py:305`);
      // completions are processed in non-decreasing `now`, so only runs of
      // equal completion time can need reordering.
      int pos = n_done++;
      while (pos > 0) {
        int prev = B.out_order[ro + pos - 1];
        if (B.b_completion[ro + prev] == now && prev > b) {
          B.out_order[ro + pos] = prev;
          pos--;
        } else {
          break;
        }
      }
      B.out_order[ro + pos] = b;
      // _colo_changed(survivors) (`simcore.py:143-146`)
      for (int i = 0; i < nrun; i++) {
        close_segment(c, slots[run[i]], run[i], now);
        reseat(c, slots, run, nrun, run[i], now);
      }
    } else {
      // ---- FORMATION: batch n_formed enters the FIFO dispatch queue
      const double t = B.b_formed[ro + n_formed];
      now = now > t ? now : t;
      n_formed++;
    }
    // ---- try_dispatch (`simcore.py:258-262`) -> GpuState.dispatch (`:153-171`)
    while (dq < n_formed && nrun < S.cap) {
      const int b = dq++;
      const int si = free_slots[--nfree];
      Slot& rb = slots[si];
      const int m = B.b_model[ro + b];
      rb.batch = b;
      rb.entry = md[m].entry_base + B.b_size[ro + b] - 1;
      rb.start = now;
      rb.total = tab.solo_ms[rb.entry];
      rb.progress = 0.0;
      rb.nseg = 0;
      rb.n_non1 = 0;
      rb.own[0] = tab.thr[3 * rb.entry + 0];
      rb.own[1] = tab.thr[3 * rb.entry + 1];
      rb.own[2] = tab.thr[3 * rb.entry + 2];
      run[nrun++] = si;
      if (B.b_running) B.b_running[ro + b] = nrun;  // dispatch trace
      reseat(c, slots, run, nrun, si, now);
      for (int i = 0; i + 1 < nrun; i++) {
        close_segment(c, slots[run[i]], run[i], now);
        reseat(c, slots, run, nrun, run[i], now);
      }
    }
  }
  if (nrun || dq < n_formed) c.status |= INTF_ST_NONQUIESCENT;
  B.n_segments[s] = seg_cursor;
  B.n_reseats[s] = c.n_reseats;
  B.status[s] = c.status;
}

// One full run_scenario for scenario s (formation + replay, no noise table).
INTF_FN void replay_scenario(int s, const intf_scenario* scens, const intf_model* models, const intf_table& tab,
                             const intf_replay_buffers& B) {
  form_scenario(s, scens, models, B);
  replay_formed(s, scens, models, tab, B);
}

// -------------------------------------------------------- features + predict
// estimate_from_history + finalize_features (`colocation.py:54-84`) and
// predict (`predict.py:43-44`, OpenBLAS ddot == fma chain) for one outcome.
INTF_FN void features_one(const double own[3], const double* colo, int nseg, int ewma, double alpha, double x[6]) {
  double r0 = colo[0], r1 = colo[1], r2 = colo[2];
  if (ewma) {
    const double om = 1.0 - alpha;
    for (int k = 1; k < nseg; k++) {
      const double* h = colo + 3 * k;
      r0 = alpha * h[0] + om * r0;  // `colocation.py:61`, two roundings + add
      r1 = alpha * h[1] + om * r1;
      r2 = alpha * h[2] + om * r2;
    }
  }
  x[0] = own[0];
  x[1] = own[1];
  x[2] = own[2];
  x[3] = r0;
  x[4] = r1;
  x[5] = r2;
}

INTF_FN double predict7(const double* w, const double x[6]) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 6; i++) acc = fma(w[i], x[i], acc);
  return acc + w[6];
}

}  // namespace intf
