// cand_stream_variants.cu -- microbenchmark (tools/, not product): work
// decomposition variants of the candidate streaming kernel (k_cand_stream)
// on the C2 shape (E = 48 own rows, ld = 20828, 32 decisions x 2 kinds,
// fp32 out = 256 MB), two output buffers alternated per launch as in bench.py.
//   v0: product shape: grid (ld/512, E, 1), 32 decisions per thread
//   v1: decisions split in 2 (grid.z = 2, 16 per thread)
//   v2: decisions split in 4 (grid.z = 4, 8 per thread)
//   v3: decisions split in 8 (grid.z = 8, 4 per thread)
//   v4: 256-thread blocks, 32 decisions per thread
//   v5: 64-thread blocks, 32 decisions per thread
//   v6: torch-like fill: one float4 per thread, huge grid
//   v7: grid-stride fill, 148 x 8 blocks of 256
//   v8: v2 with default-policy stores
//   v9/v10: decisions split in 16 / 32;  v11/v12: 256 threads, split 8 / 16
//   v13/v14: 512 threads, split 8 / 16;  v15/v16: v3/v9 with default-policy stores
//   v17: fill1 with 128-thread blocks; v18-v20: fill, J float4 per thread over a
//   contiguous block chunk (128x8, 256x4, 128x2); v21-v23: the stream kernel's
//   store pattern only (split 8 / 4 / 16); v24-v26: one kind per thread (split 8 / 4 / 16)
//   v27-v31: lockstep form (k_stream_lock) T x J = 128x2, 256x2, 128x4, 64x2, 128x1
//   v32-v35: tiled output layout (block tile contiguous), decisions split 8 / 4 / 16 / 2
//            (v32: 6.2 TB/s vs v3's 5.9 -> the product layout, csrc/predict.cu)
// Build/run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/csv2 tools/cand_stream_variants.cu && /tmp/csv2
#include <cstdio>
#include <cuda_runtime.h>

constexpr int E = 48, NDEC = 32;
constexpr long long LD = 20828;

template <int T, int DSPLIT, bool CS>
__global__ void __launch_bounds__(T) k_stream(const float* __restrict__ C0, const float* __restrict__ FE,
                                              const float4* __restrict__ coef, float* __restrict__ out) {
  constexpr int ND = NDEC / DSPLIT;
  __shared__ float4 cw[ND][2];
  const int o = blockIdx.y;
  const int d0 = blockIdx.z * ND;
  const long long r0 = ((long long)blockIdx.x * T + threadIdx.x) * 4;
  const bool inb = r0 < LD;
  const long long rr = inb ? r0 : 0;
  const float4 cx = __ldg((const float4*)(C0 + rr)), cy = __ldg((const float4*)(C0 + LD + rr)),
               cz = __ldg((const float4*)(C0 + 2 * LD + rr));
  const float4 fx = __ldg((const float4*)(FE + (o * 3 + 0) * LD + rr)),
               fy = __ldg((const float4*)(FE + (o * 3 + 1) * LD + rr)),
               fz = __ldg((const float4*)(FE + (o * 3 + 2) * LD + rr));
  for (int t = threadIdx.x; t < 2 * ND; t += T) cw[t >> 1][t & 1] = coef[((d0 + (t >> 1)) * 2 + (t & 1)) * E + o];
  __syncthreads();
  if (!inb) return;
  const long long ks = (long long)E * LD, ds = 2 * ks;
  float* row = out + ((long long)d0 * 2 * E + o) * LD + r0;
#pragma unroll 4
  for (int d = 0; d < ND; d++) {
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
    if (CS) {
      __stcs((float4*)row, yc);
      __stcs((float4*)(row + ks), yf);
    } else {
      *(float4*)row = yc;
      *(float4*)(row + ks) = yf;
    }
    row += ds;
  }
}

__global__ void k_fill1(float4* p, long long n4) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) p[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}

// fill with J float4 per thread, block chunk contiguous (thread t: base + j*T + t)
template <int T, int J>
__global__ void __launch_bounds__(T) k_fill_chunk(float4* p, long long n4) {
  const long long base = (long long)blockIdx.x * T * J;
#pragma unroll
  for (int j = 0; j < J; j++) {
    const long long i = base + (long long)j * T + threadIdx.x;
    if (i < n4) __stcs(p + i, make_float4(1.f, 1.f, 1.f, 1.f));
  }
}

// the stream kernel's store address pattern (DSPLIT decisions x 2 kinds per
// thread) with no loads and no compute
template <int T, int DSPLIT>
__global__ void __launch_bounds__(T) k_fill_pattern(float* __restrict__ out) {
  constexpr int ND = NDEC / DSPLIT;
  const int o = blockIdx.y;
  const int d0 = blockIdx.z * ND;
  const long long r0 = ((long long)blockIdx.x * T + threadIdx.x) * 4;
  if (r0 >= LD) return;
  const long long ks = (long long)E * LD, ds = 2 * ks;
  float* row = out + ((long long)d0 * 2 * E + o) * LD + r0;
  const float4 v = make_float4(1.f, 2.f, 3.f, (float)o);
#pragma unroll 4
  for (int d = 0; d < ND; d++) {
    __stcs((float4*)row, v);
    __stcs((float4*)(row + ks), v);
    row += ds;
  }
}

// kind-split stream: a thread handles one kind (3 feature loads) x ND decisions
template <int T, int DSPLIT>
__global__ void __launch_bounds__(T) k_stream_kind(const float* __restrict__ C0, const float* __restrict__ FE,
                                                   const float4* __restrict__ coef, float* __restrict__ out) {
  constexpr int ND = NDEC / DSPLIT;
  __shared__ float4 cw[ND];
  const int o = blockIdx.y;
  const int kind = blockIdx.z & 1;
  const int d0 = (blockIdx.z >> 1) * ND;
  const long long r0 = ((long long)blockIdx.x * T + threadIdx.x) * 4;
  const bool inb = r0 < LD;
  const long long rr = inb ? r0 : 0;
  const float* F = kind ? FE + (long long)o * 3 * LD : C0;
  const float4 cx = __ldg((const float4*)(F + rr)), cy = __ldg((const float4*)(F + LD + rr)),
               cz = __ldg((const float4*)(F + 2 * LD + rr));
  for (int t = threadIdx.x; t < ND; t += T) cw[t] = coef[((d0 + t) * 2 + kind) * E + o];
  __syncthreads();
  if (!inb) return;
  const long long ks = (long long)E * LD, ds = 2 * ks;
  float* row = out + ((long long)d0 * 2 * E + o) * LD + kind * ks + r0;
#pragma unroll 4
  for (int d = 0; d < ND; d++) {
    const float4 a = cw[d];
    float4 y;
    y.x = fmaf(a.z, cz.x, fmaf(a.y, cy.x, fmaf(a.x, cx.x, a.w)));
    y.y = fmaf(a.z, cz.y, fmaf(a.y, cy.y, fmaf(a.x, cx.y, a.w)));
    y.z = fmaf(a.z, cz.z, fmaf(a.y, cy.z, fmaf(a.x, cx.z, a.w)));
    y.w = fmaf(a.z, cz.w, fmaf(a.y, cy.w, fmaf(a.x, cx.w, a.w)));
    __stcs((float4*)row, y);
    row += ds;
  }
}

// lockstep form: the output of one (decision, kind) is, over the flattened
// (own, multiset) index f, ONE contiguous array (out + (d*2+k)*E*LD + 4f).  A
// CTA owns a contiguous f-range (T*J float4), loads its features once, and
// loops over the decisions; all CTAs are resident at once (one wave) and move
// through d together, so the GPU writes ~2 contiguous streams at a time.
template <int T, int J>
__global__ void __launch_bounds__(T) k_stream_lock(const float* __restrict__ C0, const float* __restrict__ FE,
                                                   const float4* __restrict__ coef, float* __restrict__ out) {
  constexpr long long L4 = LD / 4;
  __shared__ float4 cw[2][NDEC][2];
  const long long base = (long long)blockIdx.x * T * J;
  const int o_lo = (int)(base / L4);
  float4 c[J][3], f[J][3];
  int oi[J];
  bool ok[J];
#pragma unroll
  for (int j = 0; j < J; j++) {
    const long long fi = base + (long long)j * T + threadIdx.x;
    ok[j] = fi < E * L4;
    const long long fc = ok[j] ? fi : 0;
    const int o = (int)(fc / L4);
    const long long r = (fc - (long long)o * L4) * 4;
    oi[j] = o - o_lo;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      c[j][a] = __ldg((const float4*)(C0 + a * LD + r));
      f[j][a] = __ldg((const float4*)(FE + ((long long)o * 3 + a) * LD + r));
    }
  }
  for (int t = threadIdx.x; t < 2 * NDEC * 2; t += T) {
    const int w = t / (NDEC * 2), d = (t / 2) % NDEC, k = t & 1;
    const int o = min(o_lo + w, E - 1);
    cw[w][d][k] = coef[(d * 2 + k) * E + o];
  }
  __syncthreads();
  const long long ks = (long long)E * LD;
  float4* o0 = (float4*)out + base + threadIdx.x;
#pragma unroll 2
  for (int d = 0; d < NDEC; d++) {
#pragma unroll
    for (int k = 0; k < 2; k++) {
#pragma unroll
      for (int j = 0; j < J; j++) {
        const float4 w = cw[oi[j]][d][k];
        const float4* x = k ? f[j] : c[j];
        float4 y;
        y.x = fmaf(w.z, x[2].x, fmaf(w.y, x[1].x, fmaf(w.x, x[0].x, w.w)));
        y.y = fmaf(w.z, x[2].y, fmaf(w.y, x[1].y, fmaf(w.x, x[0].y, w.w)));
        y.z = fmaf(w.z, x[2].z, fmaf(w.y, x[1].z, fmaf(w.x, x[0].z, w.w)));
        y.w = fmaf(w.z, x[2].w, fmaf(w.y, x[1].w, fmaf(w.x, x[0].w, w.w)));
        if (ok[j]) __stcs(o0 + ((d * 2 + k) * ks) / 4 + j * T, y);
      }
    }
  }
}

// tiled output layout: block (x = r chunk, y = own, z = decision chunk) owns ONE
// contiguous tile [ND decisions][2 kinds][T*4 floats]; tiles ordered
// [dchunk][own][rchunk], so concurrently running blocks write adjacent tiles
template <int T, int DSPLIT>
__global__ void __launch_bounds__(T) k_stream_tiled(const float* __restrict__ C0, const float* __restrict__ FE,
                                                    const float4* __restrict__ coef, float* __restrict__ out) {
  constexpr int ND = NDEC / DSPLIT;
  __shared__ float4 cw[ND][2];
  const int o = blockIdx.y;
  const int d0 = blockIdx.z * ND;
  const long long r0 = ((long long)blockIdx.x * T + threadIdx.x) * 4;
  const bool inb = r0 < LD;
  const long long rr = inb ? r0 : 0;
  const float4 cx = __ldg((const float4*)(C0 + rr)), cy = __ldg((const float4*)(C0 + LD + rr)),
               cz = __ldg((const float4*)(C0 + 2 * LD + rr));
  const float4 fx = __ldg((const float4*)(FE + (o * 3 + 0) * LD + rr)),
               fy = __ldg((const float4*)(FE + (o * 3 + 1) * LD + rr)),
               fz = __ldg((const float4*)(FE + (o * 3 + 2) * LD + rr));
  for (int t = threadIdx.x; t < 2 * ND; t += T) cw[t >> 1][t & 1] = coef[((d0 + (t >> 1)) * 2 + (t & 1)) * E + o];
  __syncthreads();
  const long long tile = ((long long)blockIdx.z * E + o) * gridDim.x + blockIdx.x;
  float4* base = (float4*)out + tile * (ND * 2 * T) + threadIdx.x;
#pragma unroll 4
  for (int d = 0; d < ND; d++) {
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
    __stcs(base + (d * 2 + 0) * T, yc);
    __stcs(base + (d * 2 + 1) * T, yf);
  }
}

__global__ void k_fill_gs(float4* p, long long n4) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}

int main() {
  const long long out_elems = (long long)NDEC * 2 * E * LD;
  float *C0, *FE, *out[2];
  float4* coef;
  cudaMalloc(&C0, sizeof(float) * 3 * LD);
  cudaMalloc(&FE, sizeof(float) * 3 * E * LD);
  cudaMalloc(&out[0], sizeof(float) * out_elems);
  cudaMalloc(&out[1], sizeof(float) * out_elems);
  cudaMalloc(&coef, sizeof(float4) * 2 * NDEC * E);
  cudaMemset(C0, 0, sizeof(float) * 3 * LD);
  cudaMemset(FE, 0, sizeof(float) * 3 * E * LD);
  cudaMemset(coef, 0, sizeof(float4) * 2 * NDEC * E);
  const long long n4 = out_elems / 4;
  cudaEvent_t ev[64];
  for (auto& e : ev) cudaEventCreate(&e);
  auto launch = [&](int v, float* o) {
    switch (v) {
      case 0: k_stream<128, 1, true><<<dim3((LD / 4 + 127) / 128, E, 1), 128>>>(C0, FE, coef, o); break;
      case 1: k_stream<128, 2, true><<<dim3((LD / 4 + 127) / 128, E, 2), 128>>>(C0, FE, coef, o); break;
      case 2: k_stream<128, 4, true><<<dim3((LD / 4 + 127) / 128, E, 4), 128>>>(C0, FE, coef, o); break;
      case 3: k_stream<128, 8, true><<<dim3((LD / 4 + 127) / 128, E, 8), 128>>>(C0, FE, coef, o); break;
      case 4: k_stream<256, 1, true><<<dim3((LD / 4 + 255) / 256, E, 1), 256>>>(C0, FE, coef, o); break;
      case 5: k_stream<64, 1, true><<<dim3((LD / 4 + 63) / 64, E, 1), 64>>>(C0, FE, coef, o); break;
      case 6: k_fill1<<<(unsigned)((n4 + 255) / 256), 256>>>((float4*)o, n4); break;
      case 7: k_fill_gs<<<148 * 8, 256>>>((float4*)o, n4); break;
      case 8: k_stream<128, 4, false><<<dim3((LD / 4 + 127) / 128, E, 4), 128>>>(C0, FE, coef, o); break;
      case 9: k_stream<128, 16, true><<<dim3((LD / 4 + 127) / 128, E, 16), 128>>>(C0, FE, coef, o); break;
      case 10: k_stream<128, 32, true><<<dim3((LD / 4 + 127) / 128, E, 32), 128>>>(C0, FE, coef, o); break;
      case 11: k_stream<256, 8, true><<<dim3((LD / 4 + 255) / 256, E, 8), 256>>>(C0, FE, coef, o); break;
      case 12: k_stream<256, 16, true><<<dim3((LD / 4 + 255) / 256, E, 16), 256>>>(C0, FE, coef, o); break;
      case 13: k_stream<512, 8, true><<<dim3((LD / 4 + 511) / 512, E, 8), 512>>>(C0, FE, coef, o); break;
      case 14: k_stream<512, 16, true><<<dim3((LD / 4 + 511) / 512, E, 16), 512>>>(C0, FE, coef, o); break;
      case 15: k_stream<128, 8, false><<<dim3((LD / 4 + 127) / 128, E, 8), 128>>>(C0, FE, coef, o); break;
      case 16: k_stream<128, 16, false><<<dim3((LD / 4 + 127) / 128, E, 16), 128>>>(C0, FE, coef, o); break;
      case 17: k_fill1<<<(unsigned)((n4 + 127) / 128), 128>>>((float4*)o, n4); break;
      case 18: k_fill_chunk<128, 8><<<(unsigned)((n4 + 1023) / 1024), 128>>>((float4*)o, n4); break;
      case 19: k_fill_chunk<256, 4><<<(unsigned)((n4 + 1023) / 1024), 256>>>((float4*)o, n4); break;
      case 20: k_fill_chunk<128, 2><<<(unsigned)((n4 + 255) / 256), 128>>>((float4*)o, n4); break;
      case 21: k_fill_pattern<128, 8><<<dim3((LD / 4 + 127) / 128, E, 8), 128>>>(o); break;
      case 22: k_fill_pattern<128, 4><<<dim3((LD / 4 + 127) / 128, E, 4), 128>>>(o); break;
      case 23: k_fill_pattern<128, 16><<<dim3((LD / 4 + 127) / 128, E, 16), 128>>>(o); break;
      case 24: k_stream_kind<128, 8><<<dim3((LD / 4 + 127) / 128, E, 16), 128>>>(C0, FE, coef, o); break;
      case 25: k_stream_kind<128, 4><<<dim3((LD / 4 + 127) / 128, E, 8), 128>>>(C0, FE, coef, o); break;
      case 26: k_stream_kind<128, 16><<<dim3((LD / 4 + 127) / 128, E, 32), 128>>>(C0, FE, coef, o); break;
      case 27: k_stream_lock<128, 2><<<(unsigned)((n4 / NDEC / 2 + 255) / 256), 128>>>(C0, FE, coef, o); break;
      case 28: k_stream_lock<256, 2><<<(unsigned)((n4 / NDEC / 2 + 511) / 512), 256>>>(C0, FE, coef, o); break;
      case 29: k_stream_lock<128, 4><<<(unsigned)((n4 / NDEC / 2 + 511) / 512), 128>>>(C0, FE, coef, o); break;
      case 30: k_stream_lock<64, 2><<<(unsigned)((n4 / NDEC / 2 + 127) / 128), 64>>>(C0, FE, coef, o); break;
      case 31: k_stream_lock<128, 1><<<(unsigned)((n4 / NDEC / 2 + 127) / 128), 128>>>(C0, FE, coef, o); break;
      case 32: k_stream_tiled<128, 8><<<dim3((LD / 4 + 127) / 128, E, 8), 128>>>(C0, FE, coef, o); break;
      case 33: k_stream_tiled<128, 4><<<dim3((LD / 4 + 127) / 128, E, 4), 128>>>(C0, FE, coef, o); break;
      case 34: k_stream_tiled<128, 16><<<dim3((LD / 4 + 127) / 128, E, 16), 128>>>(C0, FE, coef, o); break;
      case 35: k_stream_tiled<128, 2><<<dim3((LD / 4 + 127) / 128, E, 2), 128>>>(C0, FE, coef, o); break;
    }
  };
  for (int v = 0; v < 36; v++) {
    for (int it = 0; it < 4; it++) launch(v, out[it & 1]);
    const int reps = 30;
    for (int it = 0; it < reps; it++) {
      cudaEventRecord(ev[2 * it]);
      launch(v, out[it & 1]);
      cudaEventRecord(ev[2 * it + 1]);
    }
    cudaDeviceSynchronize();
    float tot = 0.f, best = 1e9f;
    for (int it = 0; it < reps; it++) {
      float ms;
      cudaEventElapsedTime(&ms, ev[2 * it], ev[2 * it + 1]);
      tot += ms;
      best = ms < best ? ms : best;
    }
    const double mean = tot / reps;
    printf("{\"variant\": %d, \"mean_us\": %.2f, \"best_us\": %.2f, \"GBs\": %.1f, \"err\": \"%s\"}\n", v,
           mean * 1e3, best * 1e3, 4.0 * out_elems / (mean / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
