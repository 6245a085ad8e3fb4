// Batched complex128 GEMM on DMMA (mma.sync.aligned.m8n8k4.f64) for sm_100a.
// 64×64 output tile per CTA, 8 warps (2×4), warp tile 32×16, K-step 16 complex,
// cp.async double-buffered shared-memory staging with zero-fill at the edges (k4 steps past the
// end of K are skipped).  Complex product as 3 real DMMAs (P1 = ArBr, P2 = AiBi,
// P3 = (Ar+Ai)(Br+Bi); Re = P1 − P2, Im = P3 − P1 − P2), or 4 (Re += ArBr − AiBi, Im += ArBi + AiBr).
// Measured (tools/ubench_gemm.cu, B200): a 3-stage pipeline was not faster than 2 stages.
#include "gemm.cuh"

#include <algorithm>
#include <cstdlib>

namespace fmmlu {

namespace {

#ifndef FMMLU_GEMM_STAGES
#define FMMLU_GEMM_STAGES 2
#endif
constexpr int BM = 64, BN = 64, BK = 16;
constexpr int STAGES = FMMLU_GEMM_STAGES;  // cp.async pipeline depth (tiles in flight + 1)
constexpr int PADA = BM + 2, PADB = BN + 2;  // +2 complex: conflict-free fragment loads
// Tile width BN_ ∈ {64, 32}: 32 for skinny products (n ≤ 32, e.g. the multi-RHS solve sweeps), where
// a 64-wide tile would compute half zeros.  8 warps: 2×4 (warp tile 32×16) or 4×2 (16×16).
template <int BN_> struct TileCfg {
  static constexpr int WGM = BN_ == 64 ? 2 : 4, WGN = 8 / WGM;
  static constexpr int WM = BM / WGM, WN = BN_ / WGN;
  static constexpr int MI = WM / 8, NJ = WN / 8;
  static constexpr int PADB_ = BN_ + 2;
};
constexpr int NT = 256;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int src = pred ? 16 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BN_>
__device__ __forceinline__ void load_tiles(const GemmProblem& P, int m0, int n0, int k0, cplx* As,
                                           cplx* Bs, int tid) {
  constexpr int PB = TileCfg<BN_>::PADB_;
#pragma unroll
  for (int e = 0; e < (BM * BK) / NT; ++e) {
    int idx = tid + e * NT;
    int mm, kk;
    if (P.opA == kOpN) {
      mm = idx % BM;
      kk = idx / BM;
    } else {  // T or C
      kk = idx % BK;
      mm = idx / BK;
    }
    int gm = m0 + mm, gk = k0 + kk;
    bool ok = gm < P.m && gk < P.k;
    const cplx* src = ok ? (P.opA == kOpN ? P.A + gm + (size_t)gk * P.lda
                                          : P.A + gk + (size_t)gm * P.lda)
                         : P.A;
    cp_async16(&As[kk * PADA + mm], src, ok);
  }
#pragma unroll
  for (int e = 0; e < (BN_ * BK) / NT; ++e) {
    int idx = tid + e * NT;
    int nn, kk;
    if (P.opB == kOpN) {
      kk = idx % BK;
      nn = idx / BK;
    } else {  // T or C
      nn = idx % BN_;
      kk = idx / BN_;
    }
    int gn = n0 + nn, gk = k0 + kk;
    bool ok = gn < P.n && gk < P.k;
    const cplx* src = ok ? (P.opB == kOpN ? P.B + gk + (size_t)gn * P.ldb
                                          : P.B + gn + (size_t)gk * P.ldb)
                         : P.B;
    cp_async16(&Bs[kk * PB + nn], src, ok);
  }
}

template <int SCATTER, bool THREEM, int BN_ = 64>
__device__ __forceinline__ void gemm_body(const GemmProblem* __restrict__ probs,
                                          const GemmTile* __restrict__ tiles, cplx alpha,
                                          cplx* __restrict__ bsr) {
  using TC = TileCfg<BN_>;
  constexpr int MI = TC::MI, NJ = TC::NJ, PB = TC::PADB_;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* As = reinterpret_cast<cplx*>(smem_raw);      // [STAGES][BK][PADA]
  cplx* Bs = As + STAGES * BK * PADA;                // [STAGES][BK][PB]
  const GemmTile T = tiles[blockIdx.x];
  const GemmProblem P = probs[T.p];
  if (P.active != nullptr && *P.active == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / TC::WGN, wn = warp % TC::WGN;
  const int m0 = T.tm * BM, n0 = T.tn * BN_;
  const double sa = P.opA == kOpC ? -1.0 : 1.0;  // conjugation of A / B at fragment load
  const double sb = P.opB == kOpC ? -1.0 : 1.0;

  // THREEM: 3-multiplication complex product (P1 = ArBr, P2 = AiBi, P3 = (Ar+Ai)(Br+Bi);
  // Re = P1 − P2, Im = P3 − P1 − P2): 24 instead of 32 DMMAs per k-step on the tensor pipe.
  double accr[MI][NJ][2], acci[MI][NJ][2];
  double acc3[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      accr[i][j][0] = accr[i][j][1] = acci[i][j][0] = acci[i][j][1] = 0.0;
      acc3[i][j][0] = acc3[i][j][1] = 0.0;
    }

  // K range of this tile (split-K); the range is BK-aligned, P.k bounds the loads
  const int kbeg = P.kchunk > 0 ? T.ks * P.kchunk : 0;
  const int kend = P.kchunk > 0 ? min(P.k, kbeg + P.kchunk) : P.k;
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  // prologue: tiles 0 .. STAGES-2 in flight (one commit group per tile, empty groups past the end)
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_tiles<BN_>(P, m0, n0, kbeg + s * BK, As + s * BK * PADA, Bs + s * BK * PB, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();  // tile kt has landed (this thread's copies)
    __syncthreads();              // ... everybody's; and tile kt-1's buffer is free
    {
      const int kn = kt + STAGES - 1, s = kn % STAGES;
      if (kn < nk) load_tiles<BN_>(P, m0, n0, kbeg + kn * BK, As + s * BK * PADA, Bs + s * BK * PB, tid);
      cp_async_commit();
    }
    const cplx* as = As + (kt % STAGES) * BK * PADA;
    const cplx* bs = Bs + (kt % STAGES) * BK * PB;
    const int kleft = kend - (kbeg + kt * BK);  // k4 steps past the end are zero-filled: skip them
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      if (ks * 4 >= kleft) break;  // warp-uniform
      const int kk = ks * 4 + t;
      cplx a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        a[i] = as[kk * PADA + wm * TC::WM + i * 8 + g];
        a[i].y *= sa;
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        b[j] = bs[kk * PB + wn * TC::WN + j * 8 + g];
        b[j].y *= sb;
      }
      if constexpr (THREEM) {
      double as_[MI], bs_[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) as_[i] = a[i].x + a[i].y;
#pragma unroll
      for (int j = 0; j < NJ; ++j) bs_[j] = b[j].x + b[j].y;
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          dmma(accr[i][j][0], accr[i][j][1], a[i].x, b[j].x);  // P1
          dmma(acci[i][j][0], acci[i][j][1], a[i].y, b[j].y);  // P2
          dmma(acc3[i][j][0], acc3[i][j][1], as_[i], bs_[j]);  // P3
        }
      } else {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          dmma(accr[i][j][0], accr[i][j][1], a[i].x, b[j].x);
          dmma(accr[i][j][0], accr[i][j][1], a[i].y, -b[j].y);
          dmma(acci[i][j][0], acci[i][j][1], a[i].x, b[j].y);
          dmma(acci[i][j][0], acci[i][j][1], a[i].y, b[j].x);
        }
      }
    }
  }
  if constexpr (THREEM)
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double p1 = accr[i][j][h], p2 = acci[i][j][h];
        accr[i][j][h] = p1 - p2;
        acci[i][j][h] = acc3[i][j][h] - p1 - p2;
      }

  // epilogue.  Scatter: stage the tile's frame rows/columns (slot, position) and the owner-pair
  // table in shared memory (reusing the operand buffers) so each element costs 2 atomics only.
  int* rs = reinterpret_cast<int*>(smem_raw);  // [64] row slots
  int* rp = rs + BM;                           // [64] row positions
  int* cs = rp + BM;                           // [64] col slots
  int* cp = cs + BN;                           // [64] col positions
  int* bl = cp + BN;                           // [ns] block leading dims
  long long* tb = reinterpret_cast<long long*>(bl + 64);  // [ns*ns] pair offsets (if it fits)
  bool tab_in_smem = false;
  if (SCATTER) {
    tab_in_smem = P.ns <= 64 && P.ns * P.ns <= 2048;
    cp_async_wait_all();  // (only empty groups can be pending)
    __syncthreads();  // operand buffers are free
    for (int e = tid; e < BM; e += NT) {
      const int r = m0 + e;
      rs[e] = r < P.m ? P.slot[P.row0 + r] : 0;
      rp[e] = r < P.m ? P.pos[P.row0 + r] : 0;
    }
    for (int e = tid; e < BN_; e += NT) {
      const int c = n0 + e;
      cs[e] = c < P.n ? P.slot[P.col0 + c] : 0;
      cp[e] = c < P.n ? P.pos[P.col0 + c] : 0;
    }
    if (tab_in_smem) {
      for (int e = tid; e < P.ns; e += NT) bl[e] = P.bld[e];
      for (int e = tid; e < P.ns * P.ns; e += NT) tb[e] = P.tab[e];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int row = m0 + wm * TC::WM + i * 8 + g;
    if (row >= P.m) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * TC::WN + j * 8 + 2 * t + h;
        if (col >= P.n) continue;
        cplx v = cmk(alpha.x * accr[i][j][h] - alpha.y * acci[i][j][h],
                     alpha.x * acci[i][j][h] + alpha.y * accr[i][j][h]);
        if (SCATTER) {
          const int lr = row - m0, lc = col - n0;
          const int s = rs[lr], q = cs[lc];
          const long long off = tab_in_smem ? tb[s * P.ns + q] : P.tab[s * P.ns + q];
          if (off >= 0) {
            const int ld = tab_in_smem ? bl[s] : P.bld[s];
            cplx* d = bsr + off + rp[lr] + (size_t)cp[lc] * ld;
            atomicAdd(&d->x, v.x);
            atomicAdd(&d->y, v.y);
          }
        } else if (P.kchunk > 0) {
          cplx* d = P.C + row + (size_t)col * P.ldc;
          atomicAdd(&d->x, v.x);
          atomicAdd(&d->y, v.y);
        } else {
          cplx* d = P.C + row + (size_t)col * P.ldc;
          cplx c = *d;
          *d = cadd(c, v);
        }
      }
  }
}

// distinct names so profilers can tell the Schur-complement GEMM from the others
__global__ void __launch_bounds__(NT, 2) k_gemm_store(const GemmProblem* __restrict__ probs,
                                                   const GemmTile* __restrict__ tiles, cplx alpha,
                                                   cplx* __restrict__ bsr) {
  gemm_body<0, true>(probs, tiles, alpha, bsr);
}
__global__ void __launch_bounds__(NT, 2) k_gemm_store32(const GemmProblem* __restrict__ probs,
                                                     const GemmTile* __restrict__ tiles, cplx alpha,
                                                     cplx* __restrict__ bsr) {
  gemm_body<0, true, 32>(probs, tiles, alpha, bsr);
}
__global__ void __launch_bounds__(NT) k_gemm_schur(const GemmProblem* __restrict__ probs,
                                                   const GemmTile* __restrict__ tiles, cplx alpha,
                                                   cplx* __restrict__ bsr) {
  gemm_body<1, false>(probs, tiles, alpha, bsr);
}
__global__ void __launch_bounds__(NT, 2) k_gemm_schur3(const GemmProblem* __restrict__ probs,
                                                    const GemmTile* __restrict__ tiles, cplx alpha,
                                                    cplx* __restrict__ bsr) {
  gemm_body<1, true>(probs, tiles, alpha, bsr);
}

__global__ void k_gemm_expand(const GemmProblem* __restrict__ probs, const GemmGroup* __restrict__ groups,
                              int ngroups, GemmTile* __restrict__ tiles) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= ngroups) return;
  const GemmGroup g = groups[w];
  const GemmProblem& P = probs[g.p];
  const int nks = P.kchunk > 0 ? (P.k + P.kchunk - 1) / P.kchunk : 1;
  const int bn = P.bn == 32 ? 32 : BN;
  const int ntn = (P.n + bn - 1) / bn;
  for (int t = lane; t < g.count; t += 32) {
    const int ks = t % nks;
    int r = t / nks, tm = 0, tn;
    if (g.upper) {
      while (r >= ntn - tm) {
        r -= ntn - tm;
        ++tm;
      }
      tn = tm + r;
    } else {
      tm = r / ntn;
      tn = r % ntn;
    }
    tiles[g.first + t] = GemmTile{g.p, tm, tn, ks};
  }
}

}  // namespace

int gemm_tile_count(const GemmProblem& p, bool upper) {
  if (p.m <= 0 || p.n <= 0 || p.k <= 0) return 0;
  const int nks = p.kchunk > 0 ? (p.k + p.kchunk - 1) / p.kchunk : 1;
  const int bn = p.bn == 32 ? 32 : BN;
  const int tm = (p.m + BM - 1) / BM, tn = (p.n + bn - 1) / bn;
  if (!upper) return tm * tn * nks;
  int c = 0;
  for (int i = 0; i < tm; ++i) c += std::max(0, tn - i);
  return c * nks;
}

void gemm_expand(const GemmProblem* d_probs, const GemmGroup* d_groups, int ngroups, GemmTile* d_tiles,
                 cudaStream_t st) {
  if (ngroups <= 0) return;
  k_gemm_expand<<<(ngroups * 32 + 255) / 256, 256, 0, st>>>(d_probs, d_groups, ngroups, d_tiles);
  FMMLU_LAUNCH();
}

void gemm_batched(const GemmProblem* d_probs, const GemmTile* d_tiles, int ntiles, cplx alpha,
                  int scatter, cplx* bsr_base, cudaStream_t st, int bn) {
  if (ntiles <= 0) return;
  const size_t smem = (size_t)STAGES * BK * (PADA + PADB) * sizeof(cplx);
  static bool init = false;
  if (!init) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_gemm_store, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FMMLU_CUDA(cudaFuncSetAttribute(k_gemm_store32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FMMLU_CUDA(cudaFuncSetAttribute(k_gemm_schur, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FMMLU_CUDA(cudaFuncSetAttribute(k_gemm_schur3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    init = true;
  }
  // grid.x limit is 2^31-1; tiles are enumerated explicitly
  // 3-multiplication complex product in the Schur GEMM too (25 % fewer DMMAs; measured 7-10 % faster
  // on cfg5 level-5/6 shapes, tools/ubench_gemm.cu); FMMLU_SCHUR_3M=0 selects the 4-product form
  static const bool schur3 = !(getenv("FMMLU_SCHUR_3M") && atoi(getenv("FMMLU_SCHUR_3M")) == 0);
  if (scatter && schur3)
    k_gemm_schur3<<<ntiles, NT, smem, st>>>(d_probs, d_tiles, alpha, bsr_base);
  else if (scatter)
    k_gemm_schur<<<ntiles, NT, smem, st>>>(d_probs, d_tiles, alpha, bsr_base);
  else if (bn == 32)
    k_gemm_store32<<<ntiles, NT, smem, st>>>(d_probs, d_tiles, alpha, bsr_base);
  else
    k_gemm_store<<<ntiles, NT, smem, st>>>(d_probs, d_tiles, alpha, bsr_base);
  FMMLU_LAUNCH();
}

}  // namespace fmmlu
