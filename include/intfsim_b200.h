/*
 * intfsim_b200.h -- C ABI of the B200 (sm_100a) hot path of the intfsim
 * reference (arXiv 2512.18725 simulator, /root/reference/pkg/src/intfsim).
 *
 * The reference is pure Python with no FFI; its drop-in boundary is the
 * package surface `intfsim/__init__.py:7-51`.  Each entry point below is the
 * batched, device-resident replacement of one reference function (cited), and
 * is what `paper_2512_18725_b200` (the Python mirror of that surface) binds
 * with ctypes.  INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Every pointer inside the descriptor structs is a DEVICE pointer (CUDA
 *    global memory, caller-owned); the descriptor structs themselves are host
 *    memory, read during the call.  No torch types, no allocation in the hot
 *    calls: scratch comes from caller buffers.
 *  - Calls are asynchronous on `stream` (a cudaStream_t, passed as void*).
 *  - Return value: INTF_OK or an INTF_E_* code for launch/argument errors;
 *    per-scenario invariant violations (the reference's SimulationError
 *    checks, `simcore.py:118-121,155-159,175-179,302-303`) are reported in the
 *    device status word of that scenario (INTF_ST_* bit flags).
 *  - intf_last_error() returns a description of the most recent failure.
 *  - Reentrant per stream; one process per GPU for multi-GPU runs.
 */
#ifndef INTFSIM_B200_H
#define INTFSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define INTF_ABI_VERSION 1

/* return codes */
#define INTF_OK 0
#define INTF_E_BAD_INPUT 1  /* ValueError / ScenarioError / ProfileError analogue */
#define INTF_E_CUDA 2       /* CUDA launch or runtime error */
#define INTF_E_NONFINITE 3  /* PredictError (`predict.py:34-36`) */

/* device status bits, one int32 per scenario (SimulationError analogues) */
#define INTF_ST_PAST_EVENT 1      /* `simcore.py:118-121,205-206` */
#define INTF_ST_CAP 2             /* `simcore.py:155-159` */
#define INTF_ST_PROGRESS 4        /* `simcore.py:175-179` */
#define INTF_ST_NONQUIESCENT 8    /* `simcore.py:302-303` */
#define INTF_ST_OVERFLOW 16       /* a caller capacity (requests/segments) was too small: grow and retry */
#define INTF_ST_SEG_STRIDE 32     /* a batch exceeded seg_stride open segments: grow and retry */

/* Profile table (`profiles.py:18-66`): row = model_index*max_bs + (bs-1). */
typedef struct intf_table {
  const double *solo_ms; /* [n_rows] solo_duration_ms */
  const double *thr;     /* [n_rows*3] (l2, dram, sm) throughput fractions */
  int32_t n_rows, max_bs;
} intf_table;

/* One scenario (`workload.py:35-58` ScenarioSpec + `oracle.py:13-19`). */
typedef struct intf_scenario {
  int32_t n_models, model_off; /* deployed models: intf_model[model_off .. +n_models) */
  int32_t req_off, req_cap;    /* request / batch slot region */
  int32_t seg_off, seg_cap;    /* segment region */
  int32_t max_bs, cap;         /* max_batch_size, concurrency_cap */
  double duration_s, window_ms, sigma;
  double beta[3];              /* (l2, dram, sm) contention sensitivities */
  uint64_t seed, oracle_seed;  /* arrival seed, InterferenceOracle.seed */
  uint64_t batch_id_base;      /* noise key of batch b = batch_id_base + b (`oracle.py:24-33`): 0 for
                                  run_scenario; callers numbering batches across scenarios set it
                                  (full_overlap_ratios `experiments.py:266-282`) */
} intf_scenario;

/* One deployed model of a scenario (`workload.py:22-32` DeployedModel). */
typedef struct intf_model {
  int32_t entry_base;          /* table row of (model, bs=1) */
  int32_t name_rank;           /* rank of model_id among the scenario's ids in str order */
  uint32_t crc;                /* zlib crc32(model_id) (`profiles.py:239-243`) */
  int32_t list_off, list_cap;  /* per-model arrival list region */
  int32_t scen;                /* index of the owning scenario */
  double rate_rps, slo_ms;
} intf_model;

/* A batch of scenarios: descriptor arrays in device memory plus host-side
 * totals (so launches need no device->host reads). */
typedef struct intf_batch {
  const intf_scenario *scen;   /* device [n_scen] */
  const intf_model *models;    /* device [n_models] */
  int32_t n_scen, n_models;    /* totals */
  int32_t max_req_cap;         /* max over scenarios of req_cap */
  int32_t max_models;          /* max over scenarios of n_models */
  int32_t max_list_cap;        /* max over deployed models of list_cap */
  int32_t req_slots;           /* sum over scenarios of req_cap (packed request / batch slot space) */
  const int32_t *long_blocks;  /* optional device [2 * n_long_blocks]: (model, chunk) of every 256-entry
                                  chunk of every list with list_cap >= INTF_LONG_LIST, so the long-list
                                  formation launches flat grids (NULL: grids of max_list_cap x models) */
  int32_t n_long_blocks, pad_;
} intf_batch;
#ifndef INTF_LONG_LIST
#define INTF_LONG_LIST 4096 /* model lists this long form batches by chunks (and merge arrivals by time buckets) */
#endif
int intf_long_list(void); /* INTF_LONG_LIST as built (the long_blocks map must use it) */

#define INTF_SLO_WS_INTS (256 + 32 * 3 * 256 + 32 * 3 * 4)

/* Device buffers of the replay pipeline.  Index spaces:
 *   request / batch / outcome slot: req_off + i   (i < req_cap)
 *   per-model list:                 list_off + j  (j < list_cap)
 *   segment:                        seg_off + k   (k < seg_cap)      */
typedef struct intf_replay_buffers {
  double *arr_t;       /* arrival_time_ms, merged, (t, model_id) order */
  int32_t *arr_model;  /* deployed-model index */
  double *list_t;      /* per-model arrival times */
  int32_t *list_rid;   /* per-model request ids */
  int32_t *n_req;      /* [n_scen] */
  int32_t *n_list;     /* [total models] */
  int32_t *b_model, *b_size;   /* per batch id */
  double *b_formed, *b_start, *b_completion, *b_measured;
  int32_t *b_seg_off, *b_nseg; /* absolute segment index, count */
  int32_t *out_order;          /* batch id of the k-th outcome, (completion, batch_id) order */
  int32_t *b_running;          /* dispatch trace: running batches right after this batch's dispatch */
  int32_t *r_batch;            /* per request */
  uint8_t *r_slo_met;          /* per request (written by intf_slo_report) */
  double *s_tbegin, *s_tend, *s_slowdown, *s_colo; /* s_colo: [3*k] */
  int32_t *n_batches, *n_segments, *n_reseats, *status; /* [n_scen] */
  double *slot_seg;            /* scratch: n_scen*cap_max*seg_stride*5 doubles */
  double *noise_tab;           /* scratch: [req slots][noise_k] precomputed noise draws */
  double *mb_t;                /* scratch, per-model list slots: formation time of the model's c-th batch */
  int32_t *mb_info;            /* scratch, 4 per list slot: kind, key, size, head (list index of first member) */
  int32_t *n_mb;               /* scratch: [total models] batches formed per model */
  int32_t *slo_ws;             /* scratch: INTF_SLO_WS_INTS int32 for the grid-wide SLO path (long traces);
                                  slo_ws[0] is also intf_replay's scenario work counter */
  int32_t *form_ws;            /* scratch: 3 int32 per list slot, chunked formation of long lists */
  int32_t *order;              /* scratch: [n_scen + 1] replay order (longest-processing-time first) */
  int32_t seg_stride, cap_max;
  int32_t noise_k, pad_;       /* segments per batch whose noise is precomputed (0 = inline) */
} intf_replay_buffers;

/* generate_arrivals (`workload.py:74-104`): per-model Poisson streams
 * (PCG64 keyed by [seed, crc32(model)], glibc log1p), merged by
 * (t, model_id).  Fills list_t/list_rid/n_list and arr_t/arr_model/n_req.
 * `scen`, `models`: device arrays. */
int intf_generate_arrivals(const intf_batch *batch, const intf_replay_buffers *buf, void *stream);

/* Build per-model lists from caller-supplied merged arrivals (arr_t,
 * arr_model, n_req) -- for traces not produced by intf_generate_arrivals. */
int intf_split_arrivals(const intf_batch *batch, const intf_replay_buffers *buf, void *stream);

/* run_scenario (`simcore.py:218-310`): dynamic batching (`batcher.py:59-85`),
 * FIFO capped admission and reseats (`simcore.py:126-171`), noise
 * (`oracle.py:24-33`), slowdown (`oracle.py:36-47`), completion
 * (`simcore.py:56-66,173-198`), request->batch records (`:264-279`).
 * Bit-exact with the reference.  Three launches: k_form (batch formation,
 * thread per scenario), k_noise_table (the first noise_k noise draws of every
 * batch, fully parallel; skipped if noise_k == 0) and k_replay (the serial
 * admission/reseat/completion recurrence, thread per scenario). */
int intf_replay(const intf_batch *batch, const intf_table *table, const intf_replay_buffers *buf, void *stream);

/* The replay in two steps, for busy-period sharding of long traces (SURVEY
 * §8e): intf_form_batches = k_form + k_noise_table (batch ids, members,
 * formation times, noise table); intf_replay_jobs replays jobs
 * i = batches [job_lo[i], job_hi[i]) of scenario job_scen[i], each started
 * from an idle GPU, in parallel (one warp per job; slot_seg must hold
 * n_jobs*cap_max*seg_stride*5 doubles).  Outputs per batch / outcome slot are
 * exact whenever each job boundary is an idle point: the previous job of the
 * scenario must satisfy job_last_done <= b_formed[job_lo] (checked by the
 * caller, which merges failing boundaries and replays again).
 * job_info[3i..3i+2] = status bits, segment records, reseats.              */
int intf_form_batches(const intf_batch *batch, const intf_replay_buffers *buf, void *stream);
int intf_replay_jobs(const intf_batch *batch, const intf_table *table, const intf_replay_buffers *buf,
                     const int32_t *job_scen, const int32_t *job_lo, const int32_t *job_hi, int32_t n_jobs,
                     double *job_last_done, int32_t *job_info, void *stream);

/* Device-planned busy-period sharding.  Job slots of scenario s are
 * [joff[s], joff[s] + jcap[s]) (host-planned capacities; planning keeps at
 * most one job start per min_len batches, so jcap = ceil(req_cap/min_len)+1
 * suffices).  intf_jobs_plan: speculative starts (a batch forming after every
 * earlier batch's formed + slow*solo, prefix max per scenario), all jobs put
 * on the todo list (long traces: longest first).  intf_jobs_replay: replays
 * the todo list -- its first n_todo entries, or with n_todo < 0 as many as
 * todo_count[0] holds (read on the device; at most -n_todo; the warps take
 * entries from the work counter todo_count[1]), so passes queue without host
 * round trips.
 * intf_jobs_verify: per scenario, checks every boundary (previous job's last
 * completion <= first formation), merges failing ones, puts merged jobs on a
 * fresh todo list and, for scenarios whose boundaries all hold, writes the
 * per-scenario totals (n_segments, n_reseats, status).  Host loop: plan; then
 * while *todo_count: replay, reset count, verify.  The k-th todo entry of a
 * replay call uses slot_seg scratch k (size it for *todo_count jobs).      */
typedef struct intf_jobs {
  int32_t *joff, *jcap;        /* [n_scen] slot offset / capacity */
  int32_t *lo, *hi;            /* [slots] batch range of each job */
  int32_t *n_jobs;             /* [n_scen] */
  double *last;                /* [slots] last completion of the job's replay */
  int32_t *info;               /* [slots][3] status, segment records, reseats */
  uint8_t *dirty;              /* [slots] */
  int32_t *todo;               /* [slots] slots to replay */
  int32_t *todo_count;         /* [2]: [0] entries in todo, [1] intf_jobs_replay's work counter */
  int32_t *slot_scen;          /* [slots] owning scenario of each slot (host-filled) */
  double slow;                 /* optimism factor of the speculative end estimate */
  int32_t min_len, total_slots;
  double *scratch;             /* [6 * total_slots] doubles: block-parallel plan/verify of long traces
                                  (scenarios with req_cap >= 32768: one 1024-thread block each) */
  int32_t own_lo, own_hi;      /* multi-GPU sharding of one trace: intf_jobs_replay replays only jobs whose
                                  first batch lies in [own_lo, own_hi) and writes last = -inf, info = 0 for
                                  the others, so an element-wise MAX over the ranks (NCCL all_reduce) of
                                  last[] and info[] gives every rank the full job results before
                                  intf_jobs_verify; one rank: [0, INT32_MAX) */
} intf_jobs;

int intf_jobs_plan(const intf_batch *batch, const intf_table *table, const intf_replay_buffers *buf,
                   const intf_jobs *jobs, void *stream);
int intf_jobs_replay(const intf_batch *batch, const intf_table *table, const intf_replay_buffers *buf,
                     const intf_jobs *jobs, int32_t n_todo, void *stream);
int intf_jobs_verify(const intf_batch *batch, const intf_replay_buffers *buf, const intf_jobs *jobs, void *stream);

/* Per-(scenario, model) SLO report (`metrics.py:49-79`, nearest-rank
 * `percentile` `:28-36`) plus per-request slo_met (`simcore.py:268-277`).
 * warm_cutoff: device [n_scen] arrival-time cutoff or NULL (no warm-up trim).
 * Outputs indexed by model_off+m: n, met (int32), p (double[3]: p50,p95,p99). */
int intf_slo_report(const intf_batch *batch, const intf_replay_buffers *buf, const double *warm_cutoff,
                    int32_t *out_n, int32_t *out_met, double *out_p, void *stream);

/* Feature mode + linear predictor (`colocation.py:14-35`, `predict.py:26-44`). */
typedef struct intf_predictor {
  int32_t ewma;  /* 0 = static snapshot, 1 = EWMA */
  int32_t pad_;
  double alpha;  /* EWMA alpha in (0, 1] */
  double w[7];   /* w0..w5, b */
} intf_predictor;

/* samples_from_outcomes + predict (`colocation.py:95-105`, `predict.py:43-44`)
 * over replay outputs, one sample per outcome in outcome order:
 *   X[p][req_off+k][6] (f64), y[req_off+k] (f64), yhat[p][req_off+k] (f64)
 * for each of the n_pred predictors (host array).  X may be NULL. */
int intf_features_predict(const intf_batch *batch, const intf_table *table, const intf_replay_buffers *buf,
                          const intf_predictor *preds, int32_t n_pred, int64_t slot_stride, double *X, double *y,
                          double *yhat, void *stream);

/* Candidate co-location sets: every own table row x
 * every multiset of <= cap-1 peer rows, implicitly enumerated (nothing is
 * read per candidate).  For each of n_dec decisions and each candidate writes
 * the coarse (static features + coarse model) and fine (EWMA(alpha) over the
 * candidate's departure history + fine model) predicted interference ratio,
 * fp32 (fp64 features, fp32 forward: within the 1e-5 tolerance), kind 0
 * coarse, 1 fine, r < n_sets the multiset rank (size-major, colex within a
 * size), in 16 KB tiles that each streaming block writes contiguously:
 *   out[((((dec/4) * n_rows + own) * (ld/512) + r/512) * 8 + (dec%4) * 2 + kind) * 512 + r%512]
 * ld = n_sets rounded up to 512 (pad entries written as 0); the buffer holds
 * ceil(n_dec/4)*4*2*n_rows*ld floats (rows of the padded decisions unwritten).
 * coefs: device [n_dec][2][7] (w0..w5, b).                                  */
int intf_candidate_count(int32_t n_rows, int32_t cap, int64_t *n_cand, int64_t *n_sets, int64_t *ld);
/* Floats of device workspace for the two-phase form (per-(multiset, own)
 * features staged once per call -- 12 MB for the 48-row bundled table).   */
int intf_candidate_workspace(int32_t n_rows, int32_t cap, int64_t *ws_elems);
/* ws may be NULL (or too small): a single fused kernel then recomputes the
 * features in registers; with ws, k_cand_prep + k_cand_stream run.          */
int intf_predict_candidates(const intf_table *table, int32_t cap, double alpha, const double *coefs, int32_t n_dec,
                            float *out, float *ws, int64_t ws_elems, void *stream);
/* The two phases separately: features of every (multiset, own) for a
 * (table, cap, alpha) into ws (k_cand_prep), then the forward pass of n_dec
 * decisions from a prepared ws (k_cand_stream).  intf_predict_candidates
 * with ws == prepare + prepared.                                            */
int intf_candidate_prepare(const intf_table *table, int32_t cap, double alpha, float *ws, int64_t ws_elems,
                           void *stream);
int intf_predict_candidates_prepared(const intf_table *table, int32_t cap, const double *coefs, int32_t n_dec,
                                     float *out, const float *ws, int64_t ws_elems, void *stream);
/* One pipelined C2 step in a single launch (k_cand_step): the forward of
 * every candidate for coefs' n_dec decisions from the features prepared in
 * ws_cur (as intf_predict_candidates_prepared), fused with the feature build
 * for the next step into ws_next (as intf_candidate_prepare; ws_next may be
 * NULL for the last step).  ws_cur and ws_next must be distinct workspaces
 * of intf_candidate_workspace() floats.  Same reference functions as
 * intf_predict_candidates (`colocation.py:71-84`, `predict.py:43-44`). */
int intf_candidate_step(const intf_table *table, int32_t cap, double alpha, const double *coefs, int32_t n_dec,
                        float *out, const float *ws_cur, float *ws_next, int64_t ws_elems, void *stream);

/* Best candidate per (decision, kind, own row) -- what a scheduling decision
 * consumes instead of every prediction: the minimum predicted interference
 * ratio over all peer multisets of the own row, ties to the lowest multiset
 * rank, as best[(dec * 2 + kind) * n_rows + own] =
 *   (orderable fp32 bits of the value) << 32 | multiset rank
 * (orderable: v >= 0 ? bits | 1<<31 : ~bits; decode with the inverse).
 * Every candidate is still scored; only the reduction leaves the chip.
 *   intf_candidate_best_step: one pipelined step like intf_candidate_step;
 *     best must hold the all-ones key on entry (the previous step's prep
 *     blocks reset best_next for the next step); keep >= 2 key buffers and
 *     read step k's keys before step k + (buffers - 1) is launched.
 *   intf_best_candidates_host: host coefficients in, host keys out (copies
 *     on `stream`, caller synchronises); d_scratch holds 4 n_dec * 7 +
 *     4 n_dec * n_rows + the candidate workspace floats.                    */
int intf_candidate_best_step(const intf_table *table, int32_t cap, double alpha, const double *coefs, int32_t n_dec,
                             uint64_t *best, uint64_t *best_next, const float *ws_cur, float *ws_next,
                             int64_t ws_elems, void *stream);
int intf_best_candidates_host(const intf_table *table, int32_t cap, double alpha, const double *h_coefs,
                              int32_t n_dec, uint64_t *h_best, float *d_scratch, int64_t scratch_elems,
                              void *stream);
/* The host-buffer call as a pipeline of decisions: call k scores from the
 * features call k-1 built and builds call k+1's in the same launch (the
 * fused step's prep blocks), so the feature build overlaps the scoring.
 * *state counts the calls (0: build first; reset to 0 whenever table, cap or
 * alpha change); d_scratch holds intf_best_candidates_host's floats plus one
 * more candidate workspace.  With a pinned (page-locked) h_best and n_dec <=
 * 32 a call is ONE kernel launch: the coefficients travel as a kernel
 * parameter and the last block writes the keys into h_best over the bus
 * (no copies, no memset); otherwise the keys are copied back.  Either way the
 * keys are valid once the stream has synchronised.                         */
int intf_best_candidates_host_pipelined(const intf_table *table, int32_t cap, double alpha, const double *h_coefs,
                                        int32_t n_dec, uint64_t *h_best, float *d_scratch, int64_t scratch_elems,
                                        int64_t *state, void *stream);
/* The same call, synchronous: returns once the keys are in h_best.  On the
 * one-launch path (pinned h_best, n_dec <= 32) the kernel's last block also
 * writes a per-thread pinned completion word after the keys and the call
 * spins on it (no stream synchronisation); otherwise it synchronises the
 * stream.  The call a scheduler makes per decision batch.                   */
int intf_best_candidates_host_sync(const intf_table *table, int32_t cap, double alpha, const double *h_coefs,
                                   int32_t n_dec, uint64_t *h_best, float *d_scratch, int64_t scratch_elems,
                                   int64_t *state, void *stream);

/* Real scheduling decisions of a replayed batch: for every
 * batch slot (req_off + b), dec_rank = the multiset rank (enumeration of
 * cap_enum over n_rows profile rows) of the batches it co-runs with right
 * after its dispatch -- dispatched before it (FIFO) and completing strictly
 * after its start -- and dec_own = its own profile row; slots without a
 * batch get dec_rank -1.  intf_score_decisions scores every own row against
 * each decision's running set from a prepared candidate workspace
 * (intf_candidate_prepare, same cap) with one coarse / fine model
 * coefs[2][7]: best[i][2] = (orderable fp32 value << 32 | best own row),
 * chosen[i][2] = the prediction for the batch FIFO dispatched.  n_rows <= 64. */
int intf_dispatch_sets(const intf_batch *batch, const intf_replay_buffers *buf, int32_t n_rows, int32_t cap_enum,
                       int32_t *dec_rank, int32_t *dec_own, void *stream);
int intf_score_decisions(const intf_table *table, int32_t cap, const double *coefs, const float *ws, int64_t ws_elems,
                         const int32_t *dec_rank, const int32_t *dec_own, int64_t n, uint64_t *best, float *chosen,
                         void *stream);
/* The same with the EWMA candidate features in decision-major order
 * ft[r][own][3] (intf_decision_features: one transpose of a prepared
 * workspace, intf_decision_features_elems floats): a decision's 48 x 3
 * features are contiguous.                                                 */
int64_t intf_decision_features_elems(int32_t n_rows, int32_t cap);
int intf_decision_features(const intf_table *table, int32_t cap, const float *ws, int64_t ws_elems, float *ft,
                           void *stream);
int intf_score_decisions_ft(const intf_table *table, int32_t cap, const double *coefs, const float *ws,
                            int64_t ws_elems, const float *ft, const int32_t *dec_rank, const int32_t *dec_own,
                            int64_t n, uint64_t *best, float *chosen, void *stream);

/* Host-buffer variant (the end-to-end call): copies coefs in and all
 * predictions out (tiled layout above).  h_out: ceil(n_dec/4)*4*2*n_rows*ld
 * floats; d_scratch: device floats = 28*n_dec + that output size (+ the
 * workspace to use two-phase). */
int intf_predict_candidates_host(const intf_table *table, int32_t cap, double alpha, const double *h_coefs,
                                 int32_t n_dec, float *h_out, float *d_scratch, int64_t scratch_elems, void *stream);

/* OLS normal-equation statistics (`predict.py:53-66`, `rls_init` `:112-131`):
 * for n samples X[n][6] (f64), y[n] accumulate G = Z^T Z (7x7, row-major,
 * full), r = Z^T y (7), with Z = [X, 1].  out: device double[56] (G then r);
 * accumulates (+=) so several shards / ranks can be summed.  Deterministic:
 * fixed-order two-stage reduction through `ws` (INTF_OLS_WS_DOUBLES).       */
#define INTF_OLS_WS_DOUBLES (592 * 35) /* workspace for intf_ols_stats (per-block partials) */
int intf_ols_stats(const double *X, const double *y, int64_t n, double *out, double *ws, void *stream);
/* Solve the 7x7 system from stats (fp64): rank test mirroring
 * np.linalg.matrix_rank -- a condition screen on the Cholesky factor proves
 * rank 7 for well-conditioned statistics, otherwise the Gram eigenvalues --
 * ridge fallback (RIDGE_EPS=1e-8) when rank-deficient, else Cholesky.
 * out_params[7] (w0..w5, b); out_info[0] = 1 if the ridge fallback was used;
 * out_Pinv (optional, 49) = inv(Z^T Z) for rls_init.                        */
int intf_ols_solve(const double *stats, double *out_params, int32_t *out_info, double *out_Pinv, void *stream);
/* fit_ols_xy (`predict.py:53-66`) given the rows as well as their stats
 * (intf_ols_stats): as intf_ols_solve, but statistics that fail the screen
 * take matrix_rank(Z) -- and at rank 7 the solution -- from the rows: a
 * tall-skinny QR of [Z | y] by Givens rotations over the n rows (fixed merge
 * tree, deterministic) and a one-sided Jacobi SVD of R.  The Gram
 * eigenvalues cannot resolve singular values below ~sqrt(eps) S_max (exactly
 * collinear samples: a constant feature, duplicated rows), and the normal
 * equations lose cond(Z)^2 eps where lstsq (and R^-1 Q^T y) lose cond(Z) eps.
 * Well-conditioned statistics return after the screen (three launches, two
 * of them exit at once).  ws: INTF_OLS_FIT_WS_DOUBLES.                       */
#define INTF_OLS_FIT_WS_DOUBLES (128 * 35 + 8)
int intf_ols_fit_rows(const double *X, const double *y, int64_t n, const double *stats, double *ws,
                      double *out_params, int32_t *out_info, double *out_Pinv, void *stream);

/* Windowed refit ("refit each window", BASELINE configs[2]): fit_ols_xy
 * (`predict.py:53-72`) on every window of `window` consecutive rows of X
 * (n x 6, row-major) / y: n_win = ceil(n / window) fits.  stats: NULL, or
 * n_win*56 doubles that receive Z^T Z | Z^T y of every window; it is
 * required (as scratch) only for windows of > 128 rows that are not a
 * multiple of 8 (two launches).  Windows of a multiple of 8 rows with
 * 16-byte-aligned X and y are reduced and solved in one tensor-map-staged
 * launch, other windows of <= 128 rows in one thread-per-window launch;
 * params: n_win*7
 * (w0..w5, b); info: n_win*3 int32 = ridge fallback used, non-finite result
 * (PredictError), fewer than 7 rows (fit_ols raises PredictError for those;
 * fit_ols_xy solves them through the ridge fallback, as here).            */
int intf_ols_windows(const double *X, const double *y, int64_t n, int32_t window, double *stats, double *params,
                     int32_t *info, void *stream);

/* Prequential online learners (`predict.py:75-205`, `score_and_update`):
 * n_streams independent streams, stream s = samples [off[s], off[s+1]) of
 * X/y.  Each stream starts from params0[s][7] (and P0[s][49] for RLS),
 * scores each sample before updating, writes the pre-update prediction to
 * pred[i] and the final params (and P) back in place.                        */
int intf_sgd_streams(const double *X, const double *y, const int64_t *off, int32_t n_streams, const double *eta,
                     double *params, double *pred, int32_t *status, void *stream);
int intf_rls_streams(const double *X, const double *y, const int64_t *off, int32_t n_streams, const double *lam,
                     double *params, double *P, double *pred, int32_t *status, void *stream);

/* EvalReport (`predict.py:176-205`): per segment s of [off[s], off[s+1])
 * out[s][6] = (mse, rel_p25, rel_p50, rel_p75, rel_p95, n).                  */
int intf_eval_report(const double *yhat, const double *y, const int64_t *off, int32_t n_seg, double *out,
                     void *stream);

/* Per-scenario predictor evaluation of a replayed batch (SURVEY §8d C5:
 * coarse vs fine vs adaptive), composed of `experiments.py:44-60`
 * (split_samples, chronological, cut = int(round(0.75 n))), `predict.py:53-72`
 * (fit_ols), `:112-134` (rls_init with X_train), `:157-205` (evaluate,
 * score_and_update).  Scenario s has n = n_batches[s] samples in outcome order
 * at slots req_off + k of the features written by intf_features_predict:
 * X[p][slot][6] (p_static: static mode, p_ewma: EWMA mode) and y[slot].
 *   model 0 coarse   fit_ols(static[:cut]), scored offline on static[cut:]
 *   model 1 fine     fit_ols(EWMA[:cut]),   scored offline on EWMA[cut:]
 *   model 2 adaptive rls_init(fine, lam, X_train = EWMA[:cut]), prequential on EWMA[cut:]
 * params[s][3][7] (adaptive: after its tail), report[s][3][6] = (mse, rel_p25,
 * rel_p50, rel_p75, rel_p95, n_test), status[s] = 1 (fewer than 7 training
 * samples or an empty test set: the reference would raise; reports NaN, n 0)
 * | 2 coarse ridge | 4 fine ridge | 16 non-finite fit, status[S + s] = RLS bits
 * (1 non-finite, 2 P reset).  ws: intf_scenario_eval_ws(n_scen, slot_stride)
 * doubles.  Stream-ordered, no host synchronisation.                        */
int64_t intf_scenario_eval_ws(int32_t n_scen, int64_t slot_stride);
int intf_scenario_eval(const intf_batch *batch, const intf_replay_buffers *buf, const double *X, int64_t slot_stride,
                       int32_t p_static, int32_t p_ewma, const double *y, double lam, double *ws, int64_t ws_elems,
                       double *params, double *report, int32_t *status, void *stream);

/* Row-segment forms of the refit path (segment g = rows [lo[g], hi[g]) of X
 * [row][6] / y, e.g. slices of a replay's feature slots), as used by the
 * batched drift experiment (`experiments.py:153-205`):
 *   intf_ols_fit_segments  fit_ols_xy per segment (`predict.py:53-72`):
 *                          params[g][7], info[g][3] = (ridge, non-finite,
 *                          < 7 rows), Pinv[g][49] = rls_init's P0 (optional)
 *   intf_predict_segments  yhat[row] = params[model[g]] . [x, 1] (model NULL: g)
 *   intf_sgd_segments / intf_rls_segments  prequential streams over segments
 *                          (as intf_sgd_streams / intf_rls_streams)
 *   intf_eval_segments     out[g][6] EvalReport of yhat vs y over segment g;
 *                          max_len >= the longest segment.                  */
int intf_ols_fit_segments(const double *X, const double *y, const int64_t *lo, const int64_t *hi, int32_t n_seg,
                          double *params, int32_t *info, double *Pinv, void *stream);
int intf_predict_segments(const double *X, const int64_t *lo, const int64_t *hi, const int32_t *model,
                          const double *params, int32_t n_seg, double *yhat, void *stream);
int intf_sgd_segments(const double *X, const double *y, const int64_t *lo, const int64_t *hi, int32_t n_seg,
                      const double *eta, double *params, double *pred, int32_t *status, void *stream);
int intf_rls_segments(const double *X, const double *y, const int64_t *lo, const int64_t *hi, int32_t n_seg,
                      const double *lam, double *params, double *P, double *pred, int32_t *status, void *stream);
int intf_eval_segments(const double *yhat, const double *y, const int64_t *lo, const int64_t *hi, int32_t n_seg,
                       int64_t max_len, double *out, void *stream);

/* Scalar calls of the per-object API (a hand-driven GpuState, per-sample
 * learner updates): arguments as 64-bit patterns (doubles by their bits),
 * passed as kernel parameters; results written to mapped pinned memory and
 * copied to out after a stream synchronisation (one launch + one sync).
 * Same device functions and operation order as the batched entry points.
 *   NOISE    (oracle_seed, batch_id, seg_idx, sigma)   -> noise           (`oracle.py:24-33`)
 *   SLOWDOWN (own[3], colo[3], beta[3], noise)         -> slowdown        (`oracle.py:36-47`)
 *   PREDICT  (w[7], x[6])                              -> w.x + b         (`predict.py:43-44`)
 *   EWMA     (r[3], x[3], alpha)                       -> r'[3]           (`colocation.py:61`)
 *   SGD      (w[7], x[6], y, eta)                      -> w'[7], yhat, status        (`predict.py:88-95`)
 *   RLS      (w[7], P[49], x[6], y, lambda)            -> w'[7], P'[49], yhat, status (`predict.py:137-154`)
 * status: 1 non-finite parameters, 2 P reset.  Not reentrant within a host
 * thread (one mapped buffer per thread).                                    */
enum {
  INTF_SCALAR_NOISE = 0,
  INTF_SCALAR_SLOWDOWN = 1,
  INTF_SCALAR_PREDICT = 2,
  INTF_SCALAR_EWMA = 3,
  INTF_SCALAR_SGD = 4,
  INTF_SCALAR_RLS = 5
};
int intf_scalar(int32_t op, const uint64_t *args, int32_t n_args, double *out, int32_t n_out, void *stream);

/* ---- array-level entry points behind the per-object reference API ---- */

/* samples_from_outcomes over arbitrary outcome rows (`colocation.py:95-105`):
 * row i has own throughputs own[3i..3i+2], colo history colo[3*(seg_off[i]+k)]
 * for k < nseg[i]; y[i] = measured[i]/profiled[i] (`simcore.py:83-85`);
 * X[p][i][6], yhat[p][i] per predictor.  X, y, yhat may be NULL.           */
int intf_features_rows(const double *own, const int64_t *seg_off, const int32_t *nseg, const double *colo,
                       const double *measured, const double *profiled, int64_t n, const intf_predictor *preds,
                       int32_t n_pred, double *X, double *y, double *yhat, void *stream);

/* predict (`predict.py:43-44`) for rows X[n][6] and one model w[7]. */
int intf_predict_rows(const double *X, int64_t n, const double *w, double *out, void *stream);

/* nearest-rank percentiles (`metrics.py:28-36`) of values[n] at ps[nq]
 * (nq <= 8), one block, exact (radix select on IEEE bit order).            */
int intf_quantiles(const double *values, int64_t n, const double *ps, int32_t nq, double *out, void *stream);

/* slo_report over record arrays (`metrics.py:49-79`): per group g < n_groups
 * the count, met count and p50/p95/p99 of completion - arrival over records
 * with arrival >= cutoff (pass -inf for no warm-up trim).                    */
int intf_latency_report(const int32_t *group, const double *arrival, const double *completion, const uint8_t *met,
                        int64_t n, int32_t n_groups, double cutoff, int32_t *out_n, int32_t *out_met, double *out_p,
                        void *stream);

/* InterferenceOracle.noise_draw (`oracle.py:24-33`) for n keys: lognormal
 * noise of default_rng([seed, batch[i], seg[i]]), bit-exact.              */
int intf_noise_draws(uint64_t seed, double sigma, const int64_t *batch, const int64_t *seg, int64_t n, double *out,
                     void *stream);

/* oracle_slowdown (`oracle.py:36-47`) for n rows: own[3i..], colo[3i..]
 * (device), beta[3] (HOST, read at launch), noise[n] (device, or NULL = 1.0). */
int intf_slowdowns(const double *own, const double *colo, const double *beta, const double *noise, int64_t n,
                   double *out, void *stream);

/* One numpy Generator stream (SeedSequence(words) -> PCG64): n values of
 * standard_normal (uniform=0) or random() (uniform=1); serial, for pinning
 * the device RNG against numpy.                                            */
int intf_rng_stream(const uint32_t *words, int32_t n_words, int64_t n, int32_t uniform, double *out, void *stream);

/* ---- host-side CSV materialisation (no device work) ----------------------
 * The reference writes its artifacts with csv.writer rows of repr(float) /
 * int / str fields (`simcore.py:319-369` outcomes + segments, `metrics.py:
 * 82-128` requests + slo_report, `colocation.py:108-126` samples,
 * `workload.py:173-178` arrivals; writer `cli.py:34-39`).  intf_csv_rows
 * formats n_rows rows of n_cols typed SoA columns into `out` with the same
 * bytes: INTF_COL_I64 = int64 column in decimal, INTF_COL_F64_REPR = double
 * column as CPython repr(float), INTF_COL_STR = int32 indices into strtab
 * (strings already csv-quoted by the caller, lengths in strlen_tab).  Fields
 * are joined by ',' and every row ends in "\r\n".  *out_len = bytes needed;
 * out = NULL only measures.                                                  */
#define INTF_COL_I64 0
#define INTF_COL_F64_REPR 1
#define INTF_COL_STR 2
#define INTF_COL_F64_NPREPR 3 /* double column as numpy 2's repr of np.float64: "np.float64(<repr>)" */
int intf_csv_rows(int64_t n_rows, int32_t n_cols, const int32_t *kinds, const void *const *cols,
                  const char *const *strtab, const int32_t *strlen_tab, char *out, int64_t out_cap,
                  int64_t *out_len);
/* CPython repr(float) of one double into out (NUL-terminated, cap >= 32). */
int intf_repr_f64(double v, char *out, int32_t cap);

/* last error text (thread-local); returns strlen */
int intf_last_error(char *buf, int32_t n);
int intf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* INTFSIM_B200_H */
