// Microbenchmark: dependent-chain latencies of the primitives in the pivot-step kernels
// (FP64 FMA, FP64 compare+select, warp shuffle, one argmax-merge shuffle round, CTA barrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_lat tools/ubench_lat.cu
#include <cstdio>

__global__ void k(int iters, double* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999, c = 1e-9;
  long long t0, t1;
  // 1. dependent DFMA
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  // 2. dependent compare + select (argmax-merge style, FP64)
  double v = a;
  int ix = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double v2 = v * 0.5 + (double)i;
    const int i2 = ix + 1;
    if (v2 > v || (v2 == v && i2 < ix)) {
      v = v2;
      ix = i2;
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
  // 3. dependent shuffle
  int s = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
  // 4. one argmax round: shuffle (v, i) + FP64 compare + select
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, 16);
    const int i2 = __shfl_xor_sync(0xffffffffu, ix, 16);
    if (v2 > v || (v2 == v && i2 < ix)) {
      v = v2;
      ix = i2;
    }
    v += 1e-12;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
  // 5. __syncthreads (all warps)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
  // 6. __drcp_rn dependent
  double r = a;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) r = __drcp_rn(r) + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
  // 7. shared-memory store -> barrier -> load round trip
  __shared__ double sh[1024];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) sh[i & 1023] = v;
    __syncthreads();
    v = sh[i & 1023] + 1e-12;
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / iters;
  out[threadIdx.x] = a + v + s + ix + r;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* nm[7] = {"DFMA dep", "FP64 cmp+sel dep", "SHFL dep", "argmax round", "syncthreads",
                       "drcp_rn dep", "sts-bar-lds-bar"};
  for (int nt : {32, 512}) {
    k<<<1, nt>>>(1000, out, cyc);
    k<<<1, nt>>>(4000, out, cyc);
    cudaDeviceSynchronize();
    printf("threads %d:", nt);
    for (int i = 0; i < 7; ++i) printf("  %s %lld", nm[i], cyc[i]);
    printf("  (cycles)\n");
  }
  return 0;
}
