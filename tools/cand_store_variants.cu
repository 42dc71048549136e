// cand_store_variants.cu -- microbenchmark (tools/, not product): store-path
// variants of the candidate streaming kernel (k_cand_stream) on the C2 shape
// (E = 48 own rows, ld = 20828, 32 decisions x 2 kinds, fp32 out = 256 MB).
//   v0: st.global.cs (evict-first streaming stores)   -- the product kernel
//   v1: default-policy st.global.v4
//   v2: TMA bulk store: each (decision, kind) 2 KB row chunk staged in smem,
//       one thread issues cp.async.bulk.global.shared::cta (double buffered)
//   v3: fill reference (torch-like contiguous float4 stores)
// Build/run on the box: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/csv tools/cand_store_variants.cu && /tmp/csv
#include <cstdio>
#include <cuda_runtime.h>

constexpr int E = 48, NDEC = 32, T = 128;
constexpr long long LD = 20828;

template <int V>
__global__ void __launch_bounds__(T, 8) k_stream(const float* __restrict__ C0, const float* __restrict__ FE,
                                                 const float4* __restrict__ coef, float* __restrict__ out) {
  __shared__ float4 cw[NDEC][2];
  __shared__ __align__(128) float4 stage[2][2][T];  // [buf][kind][thread]
  const int o = blockIdx.y;
  const long long r0 = ((long long)blockIdx.x * T + threadIdx.x) * 4;
  const bool inb = r0 < LD;
  const long long rr = inb ? r0 : 0;
  const float4 cx = __ldg((const float4*)(C0 + rr)), cy = __ldg((const float4*)(C0 + LD + rr)),
               cz = __ldg((const float4*)(C0 + 2 * LD + rr));
  const float4 fx = __ldg((const float4*)(FE + (o * 3 + 0) * LD + rr)),
               fy = __ldg((const float4*)(FE + (o * 3 + 1) * LD + rr)),
               fz = __ldg((const float4*)(FE + (o * 3 + 2) * LD + rr));
  for (int t = threadIdx.x; t < 2 * NDEC; t += T) cw[t >> 1][t & 1] = coef[(t * E + o) % (2 * NDEC * E)];
  __syncthreads();
  const long long ks = (long long)E * LD, ds = 2 * ks;
  float* row = out + (long long)o * LD + r0;
  const long long chunk0 = (long long)o * LD + (long long)blockIdx.x * T * 4;  // block's chunk start, row (0,0)
  const int nvalid = (int)min((long long)T * 4, LD - (long long)blockIdx.x * T * 4);
  for (int d = 0; d < NDEC; d++) {
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
    if (V == 0) {
      if (inb) {
        __stcs((float4*)row, yc);
        __stcs((float4*)(row + ks), yf);
      }
    } else if (V == 1) {
      if (inb) {
        *(float4*)row = yc;
        *(float4*)(row + ks) = yf;
      }
    } else {
      const int buf = d & 1;
      if (d >= 2) {  // the bulk store issued two iterations ago must have read its buffer
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
      }
      stage[buf][0][threadIdx.x] = yc;
      stage[buf][1][threadIdx.x] = yf;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int k = 0; k < 2; k++) {
          float* g = out + chunk0 + (long long)d * ds + k * ks;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(&stage[buf][k][0]);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa),
                       "r"(nvalid * 4)
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    row += ds;
  }
  if (V == 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_fill(float4* p, long long n4) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}

int main() {
  const long long out_elems = (long long)NDEC * 2 * E * LD;
  float *C0, *FE, *out;
  float4* coef;
  cudaMalloc(&C0, sizeof(float) * 3 * LD);
  cudaMalloc(&FE, sizeof(float) * 3 * E * LD);
  cudaMalloc(&out, sizeof(float) * out_elems);
  cudaMalloc(&coef, sizeof(float4) * 2 * NDEC * E);
  cudaMemset(C0, 0, sizeof(float) * 3 * LD);
  cudaMemset(FE, 0, sizeof(float) * 3 * E * LD);
  cudaMemset(coef, 0, sizeof(float4) * 2 * NDEC * E);
  dim3 grid((unsigned)((LD / 4 + T - 1) / T), E);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](int v) {
    for (int it = 0; it < 3; it++) {
      if (v == 0) k_stream<0><<<grid, T>>>(C0, FE, coef, out);
      if (v == 1) k_stream<1><<<grid, T>>>(C0, FE, coef, out);
      if (v == 2) k_stream<2><<<grid, T>>>(C0, FE, coef, out);
      if (v == 3) k_fill<<<148 * 8, 256>>>((float4*)out, out_elems / 4);
    }
    cudaEventRecord(a);
    const int reps = 20;
    for (int it = 0; it < reps; it++) {
      if (v == 0) k_stream<0><<<grid, T>>>(C0, FE, coef, out);
      if (v == 1) k_stream<1><<<grid, T>>>(C0, FE, coef, out);
      if (v == 2) k_stream<2><<<grid, T>>>(C0, FE, coef, out);
      if (v == 3) k_fill<<<148 * 8, 256>>>((float4*)out, out_elems / 4);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double gbs = 4.0 * out_elems / (ms / 1e3) / 1e9;
    printf("{\"variant\": %d, \"us\": %.2f, \"GBs\": %.1f, \"err\": \"%s\"}\n", v, ms * 1e3, gbs,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int v = 0; v < 4; v++) run(v);
  return 0;
}
