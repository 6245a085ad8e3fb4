// Microbenchmark of the batched complex128 DMMA GEMM (paper_2201_07325_b200/csrc/gemm.cu) on
// the problem shapes of cfg5 level 6 (one colour phase): the Gram matrices G = MᴴM of the ID
// (b = 225, K = m = 7000, upper tiles), the Schur products X_{(S∪N)R}·Up (k+N = 1186, r = 60,
// scatter epilogue into a block store) and plain stores (E/F-like, m = 225, n = 1378, k = 33).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/ubench_gemm \
//        tools/ubench_gemm.cu paper_2201_07325_b200/csrc/gemm.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2201_07325_b200/csrc/gemm.cuh"

using namespace fmmlu;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__global__ void fill(cplx* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(i * 2654435761u) ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    p[i] = make_double2(((h & 0xffff) / 65536.0) - 0.5, (((h >> 16) & 0xffff) / 65536.0) - 0.5);
  }
}

struct Case {
  const char* name;
  int nprob, m, n, k, opA, opB, upper, scatter, kchunk;
};

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 5;
  std::vector<Case> cases = {
      {"gram L6 (b=225, K=7000, upper, opA=C)", 1146, 225, 225, 7000, kOpC, kOpN, 1, 0, 0},
      {"gram L7 (b=74, K=2800, upper, opA=C)", 3878, 74, 74, 2800, kOpC, kOpN, 1, 0, 0},
      {"schur L6 (kn=1186, r=60, scatter)", 1146, 1186, 1186, 60, kOpN, kOpN, 0, 1, 0},
      {"schur L5 (kn=1600, r=70, scatter)", 310, 1600, 1600, 70, kOpN, kOpN, 0, 1, 0},
      {"store E-like (m=60, n=1378, k=33, opA=T)", 1146, 60, 1378, 33, kOpT, kOpN, 0, 0, 0},
      {"store Up-like (m=60, n=1186, k=60)", 1146, 60, 1186, 60, kOpN, kOpN, 0, 0, 0},
      {"store big (m=n=4096, k=64) x4", 4, 4096, 4096, 64, kOpN, kOpN, 0, 0, 0},
  };
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  for (const Case& c : cases) {
    const size_t asz = (size_t)c.m * c.k, bsz = (size_t)c.k * c.n, csz = (size_t)c.m * c.n;
    // A and B shared by every problem (L2-resident like one box's panels), C per problem
    cplx *A, *B, *C;
    CK(cudaMalloc(&A, asz * sizeof(cplx)));
    CK(cudaMalloc(&B, bsz * sizeof(cplx)));
    const size_t cbytes = csz * c.nprob * sizeof(cplx);
    CK(cudaMalloc(&C, cbytes));
    fill<<<1024, 256>>>(A, asz, 1);
    fill<<<1024, 256>>>(B, bsz, 2);
    CK(cudaMemset(C, 0, cbytes));
    // scatter: each problem is one owner pair block of its own (ns = 1, identity frame)
    int *slot, *pos, *bld;
    long long* tab;
    CK(cudaMalloc(&slot, sizeof(int) * std::max(c.m, c.n)));
    CK(cudaMalloc(&pos, sizeof(int) * std::max(c.m, c.n)));
    CK(cudaMalloc(&bld, sizeof(int)));
    CK(cudaMalloc(&tab, sizeof(long long) * c.nprob));
    {
      std::vector<int> z(std::max(c.m, c.n), 0), p(std::max(c.m, c.n));
      for (size_t i = 0; i < p.size(); ++i) p[i] = (int)i;
      CK(cudaMemcpy(slot, z.data(), z.size() * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(pos, p.data(), p.size() * sizeof(int), cudaMemcpyHostToDevice));
      int l = c.m;
      CK(cudaMemcpy(bld, &l, sizeof(int), cudaMemcpyHostToDevice));
      std::vector<long long> t(c.nprob);
      for (int i = 0; i < c.nprob; ++i) t[i] = (long long)i * csz;
      CK(cudaMemcpy(tab, t.data(), t.size() * sizeof(long long), cudaMemcpyHostToDevice));
    }
    std::vector<GemmProblem> probs(c.nprob);
    std::vector<GemmGroup> groups;
    long long ntiles = 0;
    for (int i = 0; i < c.nprob; ++i) {
      GemmProblem& P = probs[i];
      P = GemmProblem{};
      P.m = c.m;
      P.n = c.n;
      P.k = c.k;
      P.opA = c.opA;
      P.opB = c.opB;
      P.A = A;
      P.lda = c.opA == kOpN ? c.m : c.k;
      P.B = B;
      P.ldb = c.opB == kOpN ? c.k : c.n;
      P.C = C + (size_t)i * csz;
      P.ldc = c.m;
      P.kchunk = c.kchunk;
      if (c.scatter) {
        P.ns = 1;
        P.slot = slot;
        P.pos = pos;
        P.bld = bld;
        P.tab = tab + i;
      }
      const int cnt = gemm_tile_count(P, c.upper);
      groups.push_back(GemmGroup{i, (int)ntiles, cnt, c.upper});
      ntiles += cnt;
    }
    GemmProblem* dP;
    GemmGroup* dG;
    GemmTile* dT;
    CK(cudaMalloc(&dP, probs.size() * sizeof(GemmProblem)));
    CK(cudaMalloc(&dG, groups.size() * sizeof(GemmGroup)));
    CK(cudaMalloc(&dT, ntiles * sizeof(GemmTile)));
    CK(cudaMemcpy(dP, probs.data(), probs.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dG, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    gemm_expand(dP, dG, (int)groups.size(), dT, st);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    gemm_batched(dP, dT, (int)ntiles, make_double2(-1.0, 0.0), c.scatter, C, st);  // warm-up
    CK(cudaStreamSynchronize(st));
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(e0, st));
      gemm_batched(dP, dT, (int)ntiles, make_double2(-1.0, 0.0), c.scatter, C, st);
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    const double fl = 8.0 * c.m * (double)c.n * c.k * c.nprob * (c.upper ? 0.5 : 1.0);
    printf("%-44s tiles %8lld  %8.3f ms  %6.2f TFLOP/s (algorithmic)\n", c.name, ntiles, best, fl / best / 1e9);
    CK(cudaFree(A));
    CK(cudaFree(B));
    CK(cudaFree(C));
    CK(cudaFree(slot));
    CK(cudaFree(pos));
    CK(cudaFree(bld));
    CK(cudaFree(tab));
    CK(cudaFree(dP));
    CK(cudaFree(dG));
    CK(cudaFree(dT));
  }
  return 0;
}
