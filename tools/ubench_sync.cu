// Microbenchmark: per-step cost of the synchronisation patterns used by the register-resident
// Gauss-Jordan kernel (cluster barrier, CTA barrier, L2 exchange), 512 threads per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ubench_sync tools/ubench_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int steps, double2* x, int* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double2 sh[1024];
  int acc = 0;
  double2 v = make_double2(0, 0);
  for (int j = 0; j < steps; ++j) {
    if (MODE == 0) {  // cluster barrier only
      cl.sync();
    } else if (MODE == 1) {  // CTA barrier only
      __syncthreads();
    } else if (MODE == 2) {  // cluster barrier + CTA barrier
      cl.sync();
      __syncthreads();
    } else if (MODE == 3) {  // owner writes 512 values to global, cluster barrier, all read them (L2)
      double2* b = x + (size_t)blockIdx.y * 2048 + (j & 1) * 1024;
      if (cl.block_rank() == (unsigned)(j % cl.num_blocks())) b[threadIdx.x] = make_double2(j, threadIdx.x);
      cl.sync();
      double2 r = __ldcg(b + threadIdx.x);
      v.x += r.x;
      __syncthreads();
    } else if (MODE == 4) {  // same through DSMEM
      const unsigned o = j % cl.num_blocks();
      if (cl.block_rank() == o) sh[(j & 1) * 512 + threadIdx.x] = make_double2(j, threadIdx.x);
      cl.sync();
      const double2* rb = cl.map_shared_rank(sh + (j & 1) * 512, o);
      v.x += rb[threadIdx.x].x;
      __syncthreads();
    }
    acc += j;
  }
  cl.sync();  // no CTA exits while others may still read its shared memory
  if (threadIdx.x == 0) out[blockIdx.x] = acc + (int)v.x;
}

template <int MODE>
float run(int CL, int ny, int steps, double2* x, int* out) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL, ny, 1);
  cfg.blockDim = dim3(512, 1, 1);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (CL > 8) cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaError_t e0 = cudaLaunchKernelEx(&cfg, k<MODE>, steps, x, out);
  if (e0 != cudaSuccess) {
    printf("launch error %s (CL %d)\n", cudaGetErrorString(e0), CL);
    fflush(stdout);
    return -1.f;
  }
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k<MODE>, steps, x, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / steps;  // µs per step
}

int main() {
  double2* x;
  int* out;
  setvbuf(stdout, nullptr, _IONBF, 0);
  cudaMalloc(&x, 64 * 2048 * sizeof(double2));
  cudaMalloc(&out, 4096 * sizeof(int));
  const int steps = 4000;
  for (int CL : {1, 2, 4, 8, 16})
    for (int ny : {1, 8}) {
      printf("CL %2d ny %d: cl.sync %.3f us  syncthreads %.3f us  both %.3f us  L2-xchg %.3f us  DSMEM-xchg %.3f us\n",
             CL, ny, run<0>(CL, ny, steps, x, out), run<1>(CL, ny, steps, x, out), run<2>(CL, ny, steps, x, out),
             run<3>(CL, ny, steps, x, out), run<4>(CL, ny, steps, x, out));
    }
  return 0;
}
