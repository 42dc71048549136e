// hostcheck.cpp -- TEST-ONLY host build of the product's replay logic.
//
// Compiles paper_2512_18725_b200/csrc/replay_core.cuh with g++
// (-DINTF_HOST_CHECK -ffp-contract=off) so tests/ can exercise the exact
// recurrence the sm_100a kernels run, against the oracle, on a machine
// without a GPU.  It mirrors k_gen_arrivals / k_merge_arrivals / k_replay /
// k_features one-for-one.  Never shipped or loaded by the product.
#define INTF_HOST_CHECK 1
#include "../../paper_2512_18725_b200/csrc/replay_core.cuh"

using namespace intf;

extern "C" int hc_run(const intf_batch* bt, const intf_table* tab, const intf_replay_buffers* B, int gen) {
  const int S_n = bt->n_scen;
  if (gen) {
    for (int s = 0; s < S_n; s++) { B->n_req[s] = 0; B->status[s] = 0; }
    for (int g = 0; g < bt->n_models; g++) {
      const intf_model& M = bt->models[g];
      int n = gen_model_arrivals(bt->scen[M.scen], M, B->list_t + M.list_off, M.list_cap);
      if (n > M.list_cap) B->status[M.scen] |= INTF_ST_OVERFLOW;
      B->n_list[g] = n;
      B->n_req[M.scen] += n;
    }
    for (int g = 0; g < bt->n_models; g++) {
      const intf_model& M = bt->models[g];
      const intf_scenario& S = bt->scen[M.scen];
      if (B->status[M.scen] & INTF_ST_OVERFLOW) continue;
      int n = B->n_list[g];
      for (int j = 0; j < n; j++) {
        double t = B->list_t[M.list_off + j];
        int pos = j;
        for (int q = 0; q < S.n_models; q++) {
          int gq = S.model_off + q;
          if (gq == g) continue;
          const intf_model& Q = bt->models[gq];
          pos += count_before(B->list_t + Q.list_off, B->n_list[gq], t, Q.name_rank < M.name_rank);
        }
        B->list_rid[M.list_off + j] = pos;
        B->arr_t[S.req_off + pos] = t;
        B->arr_model[S.req_off + pos] = g - S.model_off;
      }
    }
  }
  for (int s = 0; s < S_n; s++) {
    if (B->status[s] & INTF_ST_OVERFLOW) {
      B->n_batches[s] = 0;
      continue;
    }
    form_scenario(s, bt->scen, bt->models, *B);
  }
  for (int s = 0; s < S_n; s++) {  // mirrors k_noise_table
    const intf_scenario& S = bt->scen[s];
    for (int b = 0; b < B->n_batches[s]; b++)
      for (int k = 0; k < B->noise_k; k++)
        B->noise_tab[(long long)(S.req_off + b) * B->noise_k + k] = noise_draw(S.oracle_seed, S.batch_id_base + b, k, S.sigma);
  }
  for (int s = 0; s < S_n; s++) {
    if (B->status[s] & INTF_ST_OVERFLOW) continue;
    replay_formed(s, bt->scen, bt->models, *tab, *B);
  }
  return 0;
}

extern "C" void hc_features(const intf_batch* bt, const intf_table* tab, const intf_replay_buffers* B,
                            const intf_predictor* P, int n_pred, long long stride, double* X, double* Y, double* Yh) {
  for (int s = 0; s < bt->n_scen; s++) {
    const intf_scenario& S = bt->scen[s];
    for (int k = 0; k < B->n_batches[s]; k++) {
      long long slot = (long long)S.req_off + k;
      int b = B->out_order[slot];
      long long bs = (long long)S.req_off + b;
      int entry = bt->models[S.model_off + B->b_model[bs]].entry_base + B->b_size[bs] - 1;
      double own[3] = {tab->thr[3 * entry], tab->thr[3 * entry + 1], tab->thr[3 * entry + 2]};
      Y[slot] = B->b_measured[bs] / tab->solo_ms[entry];
      for (int p = 0; p < n_pred; p++) {
        double x[6];
        features_one(own, B->s_colo + 3ll * B->b_seg_off[bs], B->b_nseg[bs], P[p].ewma, P[p].alpha, x);
        for (int i = 0; i < 6; i++) X[(p * stride + slot) * 6 + i] = x[i];
        Yh[p * stride + slot] = predict7(P[p].w, x);
      }
    }
  }
}

extern "C" double hc_noise(unsigned long long seed, unsigned b, unsigned k, double sigma) {
  return noise_draw(seed, b, k, sigma);
}
// noise_draws_k (the noise table's shared-prefix form) vs noise_draw per
// draw: mismatching draws counted over n (seed, batch) pairs x K segments
extern "C" long long hc_noise_k_mismatch(const unsigned long long* seed, const unsigned long long* batch, long long n,
                                         int K, double sigma) {
  long long bad = 0;
  double out[16];
  for (long long i = 0; i < n; i++) {
    noise_draws_k(seed[i], batch[i], K, sigma, out);
    for (int j = 0; j < K; j++) bad += out[j] != noise_draw(seed[i], batch[i], (uint64_t)j, sigma);
  }
  return bad;
}
extern "C" double hc_exp(double x) { return glibc_exp(x); }
extern "C" double hc_log1p(double x) { return glibc_log1p(x); }
