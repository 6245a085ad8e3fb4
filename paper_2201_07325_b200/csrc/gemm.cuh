// Batched variable-size complex128 GEMM on the FP64 tensor path (DMMA
// mma.sync.m8n8k4.f64 — tcgen05 has no f64 kind), with two
// epilogues:
//   kStore      : C = C + alpha * op(A) op(B)                  (E/F transforms, LU updates)
//   kScatterAdd : Δ[(S∪N) frame] += alpha * op(A) op(B), scattered with fp64 atomics
//                 into the level's block-sparse "current matrix" store (the Schur
//                 complement update −X_{(S∪N)R} X_RR⁻¹ X_{R(S∪N)}, PAPER.md L676-680,
//                 L813-825).
#pragma once
#include "common.cuh"

namespace fmmlu {

enum : int { kOpN = 0, kOpT = 1, kOpC = 2 };  // C = conjugate transpose

struct GemmProblem {
  int m, n, k;
  int opA, opB;
  int lda, ldb, ldc;
  const cplx* A;
  const cplx* B;
  cplx* C;  // kStore: C itself; kScatterAdd: unused
  // scatter epilogue: output row i (col j) of the problem maps to frame index
  // row0 + i (col0 + j); frame index f -> (slot[f], pos[f]); block pointer for
  // slot pair (s, t) is tab[s * ns + t] (complex offset into the BSR arena, -1 = absent),
  // block leading dimension is ld[s].
  int row0, col0, ns;
  const int* slot;
  const int* pos;
  const long long* tab;
  const int* bld;
  int kchunk;  // split-K: each tile covers K range [ks*kchunk, (ks+1)*kchunk); 0 = whole K.
               // With split-K the kStore epilogue accumulates with fp64 atomics.
  const int* active;  // optional device flag: tile is skipped when *active == 0
  int bn;             // output tile width: 32 (skinny n ≤ 32 stores) or 64 (0 = 64)
};

struct GemmTile {
  int p;   // problem index
  int tm;  // tile row
  int tn;  // tile col
  int ks;  // K split index
};

// C = C + alpha * op(A) op(B) for each problem; `tiles` enumerates 64×64 output tiles.
void gemm_batched(const GemmProblem* d_probs, const GemmTile* d_tiles, int ntiles, cplx alpha,
                  int scatter, cplx* bsr_base, cudaStream_t st, int bn = 64);

// Compact host description of a problem's tiles: tiles [first, first + count) of the launch belong
// to problem p (upper = 1: only tile rows ≤ tile columns, Hermitian results).  The per-tile list is
// expanded on the device (one warp per group), so the host never enumerates tiles.
struct GemmGroup {
  int p, first, count, upper;
};
int gemm_tile_count(const GemmProblem& p, bool upper);
void gemm_expand(const GemmProblem* d_probs, const GemmGroup* d_groups, int ngroups, GemmTile* d_tiles,
                 cudaStream_t st);

}  // namespace fmmlu
