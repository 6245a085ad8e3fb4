// Root block of the factorization (the actives B_t left after level 2 form a
// dense block that is factored by "dense LU"): blocked right-looking LU with partial pivoting,
// P A = L U (L unit lower, U upper, LAPACK getrf pivot convention), and the triangular solves /
// products that the solve, the forward apply and the multi-RHS sweeps use.
//
//   for each outer panel J = [J0, J0+NB):                                  (NB = kRootNB)
//     for each inner panel [j0, j0+jb) ⊂ J:                                 (jb = kRootIB)
//       k_lu_panel      rows j0..n-1 × the jb panel columns, register-resident over a 16-CTA
//                       cluster: pivot search (argmax |a_ij|, ties → lowest row), interchange,
//                       multipliers l_ij = a_ij / u_jj, rank-1 updates inside the panel
//       k_lu_swap_trsm  the jb interchanges on the other columns of J, U12 = L11⁻¹ A12 on J's
//                       columns right of the panel
//       DMMA GEMM       A[j0+jb:, right part of J] −= L21 · U12
//     k_lu_swap_trsm    the NB interchanges on every column outside J, U12 = L11⁻¹ A12 right of J
//     DMMA GEMM         trailing update A[J0+NB:, J0+NB:] −= L21 · U12       (8/3·n³ flops total)
//   k_lu_diag_inv       inverses of the kRootTB×kRootTB diagonal blocks of L and U (solve helpers)
//
// Solve (y ← U⁻¹ L⁻¹ P y): sync-free blocked triangular solves, one CTA per kRootTB-row block
// taking blocks in dependency order from an atomic ticket (so every block it waits on is already
// running); a block subtracts the off-diagonal tiles of the blocks published before it, applies
// its diagonal-block inverse and publishes its rows with a release flag.
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include <climits>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fmmlu {

namespace {

constexpr int LU_NT = 512, LU_NW = LU_NT / 32, LU_RMAX = 512;  // rows per CTA ≤ 16 row groups × 32
constexpr int LU_CL = 16;                                       // CTAs per cluster (rows split)
constexpr int LU_JB = 32;                                       // widest panel

__device__ __forceinline__ void lu_argmax(double& v, int& idx) {
  const unsigned long long key = v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const unsigned bi = __reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)idx : 0xffffffffu);
  idx = (int)bi;
  v = idx == INT_MAX ? -1.0 : __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
}

// Panel LU of rows [j0, n) × columns [j0, j0+jb) of A (ld lda), jb ≤ MC·CG ≤ 64.  Rows are split
// over the CL CTAs of the cluster (CTA c: local rows [c·rc, (c+1)·rc) of the trailing block); jb ≤ 32;
// inside a CTA warp (rg, cgp) holds row rg·32 + lane and panel columns cgp + CG·q (q < MC) in
// registers.  Per column s (pivot row j = j0 + s):
//   P1  the warps of column s publish its values and per-warp argmax candidates (rows ≥ j)
//   P2  the CTA winner's row and (owner) the current row j are pushed into every CTA's shared
//       memory with the candidate; ONE cluster barrier; every warp reduces the CL candidates → p
//   P3  rows j and p are interchanged; rows below j: l = a_is / u_js, a_ic −= l u_jc (c > s)
// piv[j] = p (global row of the n-row block).  An exactly zero pivot column sets *status.
template <int MC>
__global__ void __launch_bounds__(LU_NT, 1) k_lu_panel(cplx* __restrict__ A, int lda, int n, int* __restrict__ piv,
                                                       int j0, int jb, int* status) {
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  __shared__ cplx crow[2][LU_CL][LU_JB];  // every CTA's candidate row (pushed), [parity][rank][col]
  __shared__ cplx cold[2][LU_JB];         // current row j (pushed by its owner)
  __shared__ double ccv[2][LU_CL];
  __shared__ int cci[2][LU_CL];
  __shared__ double wcv[2][LU_NW];
  __shared__ int wci[2][LU_NW];
  __shared__ cplx fcol[2][LU_RMAX];
  __shared__ cplx mrow[LU_JB], mold[LU_JB];
  const int nr = n - j0;
  const int rc = (nr + CL - 1) / CL;
  const int r0 = j0 + rank * rc, r1 = min(n, r0 + rc);
  const int RG = (rc + 31) >> 5, CG = LU_NW / RG;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rg = warp % RG, cgp = warp / RG;
  if ((jb + CG - 1) / CG > MC || RG > LU_NW || jb > LU_JB || CL > LU_CL) __trap();  // configuration mismatch
  const int nq = cgp < CG ? min(MC, (jb - cgp + CG - 1) / CG) : 0;
  const int il = rg * 32 + lane;
  const int i = r0 + il;
  const bool rowok = il < rc && i < r1;
  cplx a[MC];
#pragma unroll
  for (int q = 0; q < MC; ++q) {
    const int c = cgp + CG * q;
    a[q] = (q < nq && rowok) ? A[i + (size_t)(j0 + c) * lda] : cmk(0.0, 0.0);
  }
  for (int s = 0; s < jb; ++s) {
    const int j = j0 + s, par = s & 1;
    if (cgp < CG && cgp == s % CG) {  // P1: column s
      const int qs = s / CG;
      cplx x = a[0];
#pragma unroll
      for (int q = 1; q < MC; ++q)
        if (q == qs) x = a[q];
      if (rowok) fcol[par][il] = x;
      double v = (rowok && i >= j) ? cabs2(x) : -1.0;
      int ix = (rowok && i >= j) ? i : INT_MAX;
      lu_argmax(v, ix);
      if (lane == 0) {
        wcv[par][rg] = v;
        wci[par][rg] = ix;
      }
    }
    __syncthreads();
    double lv = lane < RG ? wcv[par][lane] : -1.0;
    int li = lane < RG ? wci[par][lane] : INT_MAX;
    lu_argmax(lv, li);
    if (rowok && (i == li || i == j)) {
#pragma unroll
      for (int q = 0; q < MC; ++q) {
        if (q >= nq) break;
        const int c = cgp + CG * q;
        if (i == li) mrow[c] = a[q];
        if (i == j) mold[c] = a[q];
      }
    }
    __syncthreads();
    const bool ownj = j >= r0 && j < r1;
    for (int e = tid; e < CL * jb; e += LU_NT) {  // P2: push
      const int dst = e / jb, c = e - dst * jb;
      *cl.map_shared_rank(&crow[par][rank][c], dst) = mrow[c];
      if (ownj) *cl.map_shared_rank(&cold[par][c], dst) = mold[c];
    }
    if (tid < CL) {
      *cl.map_shared_rank(&ccv[par][rank], tid) = lv;
      *cl.map_shared_rank(&cci[par][rank], tid) = li;
    }
    cl.sync();
    double pv = lane < CL ? ccv[par][lane] : -1.0;
    int p = lane < CL ? cci[par][lane] : INT_MAX;
    lu_argmax(pv, p);
    const bool sing = !(pv > 0.0) || p == INT_MAX;
    if (sing) p = j;
    const int po = (p - j0) / rc;
    if (rank == 0 && tid == 0) {
      piv[j] = p;
      if (sing) atomicExch(status, 1);
    }
    const cplx* const orow = cold[par];
    const cplx* const prow = sing ? orow : crow[par][po];
    const cplx d = prow[s];
    const double rn = sing ? 0.0 : __drcp_rn(d.x * d.x + d.y * d.y);
    const cplx dinv = cmk(d.x * rn, -d.y * rn);
    if (rowok && i >= j) {  // P3 (rows above j are final)
      const bool isj = i == j, isp = i == p && p != j;
      const cplx f = isp ? orow[s] : fcol[par][il];
      const cplx l = cmul(f, dinv);
#pragma unroll
      for (int q = 0; q < MC; ++q) {
        if (q >= nq) break;
        const int c = cgp + CG * q;
        if (isj) {
          a[q] = prow[c];
        } else {
          const cplx old = isp ? orow[c] : a[q];
          a[q] = c < s ? old : (c == s ? l : cfms(l, prow[c], old));
        }
      }
    }
  }
  cl.sync();  // no CTA exits while others may still push into its shared memory
#pragma unroll
  for (int q = 0; q < MC; ++q) {
    if (q >= nq || !rowok) break;
    const int c = cgp + CG * q;
    A[i + (size_t)(j0 + c) * lda] = a[q];
  }
}

// The interchanges piv[j0 .. j0+jb) (applied in order) on columns [c_lo, c_hi) outside
// [skip_lo, skip_hi), composed into one permutation of the ≤ 2 jb affected rows and applied as a
// gather; then, on columns ≥ trsm_from, rows [j0, j0+jb) ← L11⁻¹ · rows [j0, j0+jb) (L11 = the unit
// lower jb × jb block at (j0, j0)).  One CTA per SW_C columns.
constexpr int SW_C = 32, SW_NT = 256;
__global__ void __launch_bounds__(SW_NT) k_lu_swap_trsm(cplx* __restrict__ A, int lda, int n,
                                                        const int* __restrict__ piv, int j0, int jb, int c_lo,
                                                        int c_hi, int skip_lo, int skip_hi, int trsm_from) {
  extern __shared__ __align__(16) unsigned char sw_sh[];
  cplx* L11 = reinterpret_cast<cplx*>(sw_sh);                        // [jb][jb] (column-major)
  cplx* vals = L11 + (size_t)jb * jb;                                // [SW_C][2 jb]
  int* rows = reinterpret_cast<int*>(vals + (size_t)SW_C * 2 * jb);  // [2 jb] affected rows
  int* mp = rows + 2 * jb;                                           // [n] row → source row (affected only)
  __shared__ int nr_s;
  const int c0 = c_lo + blockIdx.x * SW_C;
  if (threadIdx.x == 0) {
    int nr = 0;
    for (int s = 0; s < jb; ++s) {
      mp[j0 + s] = -1;
      mp[piv[j0 + s]] = -1;
    }
    for (int s = 0; s < jb; ++s) {
      const int j = j0 + s, p = piv[j];
      if (mp[j] < 0) { mp[j] = j; rows[nr++] = j; }
      if (mp[p] < 0) { mp[p] = p; rows[nr++] = p; }
    }
    for (int s = 0; s < jb; ++s) {  // row j ↔ row p, in order: mp[r] = original row now in r
      const int j = j0 + s, p = piv[j];
      const int t = mp[j];
      mp[j] = mp[p];
      mp[p] = t;
    }
    nr_s = nr;
  }
  const bool do_trsm = trsm_from < n && c0 + SW_C > trsm_from;
  if (do_trsm)
    for (int e = threadIdx.x; e < jb * jb; e += SW_NT) L11[e] = A[(j0 + e % jb) + (size_t)(j0 + e / jb) * lda];
  __syncthreads();
  const int nr = nr_s;
  for (int e = threadIdx.x; e < SW_C * nr; e += SW_NT) {
    const int k = e % nr, cl = e / nr, c = c0 + cl;
    if (c < c_hi && !(c >= skip_lo && c < skip_hi)) vals[cl * 2 * jb + k] = A[mp[rows[k]] + (size_t)c * lda];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < SW_C * nr; e += SW_NT) {
    const int k = e % nr, cl = e / nr, c = c0 + cl;
    if (c < c_hi && !(c >= skip_lo && c < skip_hi)) A[rows[k] + (size_t)c * lda] = vals[cl * 2 * jb + k];
  }
  if (!do_trsm) return;
  __syncthreads();
  // forward substitution, 8 threads per column: thread (cl, g) owns rows s ≡ g (mod 8)
  const int cl = threadIdx.x >> 3, g = threadIdx.x & 7, c = c0 + cl;
  const bool ok = c < c_hi && c >= trsm_from && !(c >= skip_lo && c < skip_hi);
  cplx* x = vals + (size_t)cl * 2 * jb;  // reuse as the column's jb values
  if (ok)
    for (int s = g; s < jb; s += 8) x[s] = A[(j0 + s) + (size_t)c * lda];
  __syncwarp();
  for (int s = 0; s < jb; ++s) {
    const cplx xs = x[s];  // final once every t < s has been subtracted
    __syncwarp();
    if (ok)
      for (int r = s + 1 + ((g - (s + 1)) & 7); r < jb; r += 8) x[r] = cfms(L11[r + (size_t)s * jb], xs, x[r]);
    __syncwarp();
  }
  if (ok)
    for (int s = g; s < jb; s += 8) A[(j0 + s) + (size_t)c * lda] = x[s];
}

// Inverses of the TB × TB diagonal blocks of L (unit lower) and U (upper): Dinv holds, per block b,
// Linv_b (TB × TB, column-major) then Uinv_b.  One CTA per (block, factor); column-by-column
// substitution in shared memory (TB ≤ 64).
__global__ void __launch_bounds__(256) k_lu_diag_inv(const cplx* __restrict__ A, int lda, int n, int TB,
                                                     cplx* __restrict__ Dinv) {
  extern __shared__ __align__(16) unsigned char dv_sh[];
  cplx* M = reinterpret_cast<cplx*>(dv_sh);  // [TB][TB] block
  cplx* X = M + TB * TB;                     // [TB][TB] inverse
  const int b = blockIdx.x, upper = blockIdx.y;
  const int o = b * TB, m = min(TB, n - o);
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    const int r = e % TB, c = e / TB;
    M[e] = (r < m && c < m) ? A[(o + r) + (size_t)(o + c) * lda] : cmk(r == c ? 1.0 : 0.0, 0.0);
    X[e] = cmk(0.0, 0.0);
  }
  __syncthreads();
  // column c of the inverse: solve M x = e_c (lower: forward, unit diagonal; upper: backward)
  for (int c = threadIdx.x; c < TB; c += blockDim.x) {
    cplx* x = X + (size_t)c * TB;
    if (!upper) {
      x[c] = cmk(1.0, 0.0);
      for (int s = c; s < TB; ++s) {
        const cplx xs = x[s];
        for (int r = s + 1; r < TB; ++r) x[r] = cfms(M[r + (size_t)s * TB], xs, x[r]);
      }
    } else {
      for (int s = c; s >= 0; --s) {
        cplx v = s == c ? cmk(1.0, 0.0) : cmk(0.0, 0.0);
        for (int t = s + 1; t <= c; ++t) v = cfms(M[s + (size_t)t * TB], x[t], v);
        const cplx d = M[s + (size_t)s * TB];
        const double rn = 1.0 / cabs2(d);
        x[s] = cmul(v, cmk(d.x * rn, -d.y * rn));
      }
    }
  }
  __syncthreads();
  cplx* out = Dinv + ((size_t)b * 2 + upper) * TB * TB;
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) out[e] = X[e];
}

// Blocked triangular solve on Y (n × nq, ld ldy, nq ≤ TS_Q) with the LU in A: lower (unit L,
// forward) or upper (U, backward).  Blocks of TB rows; a CTA takes the next block in dependency
// order from *ticket, subtracts M[rows, cols of every earlier block] · Y[those rows] as soon as
// that block's flag is released, multiplies by its diagonal-block inverse, writes its rows and
// releases its flag.  flags[nblk] and *ticket must be zero at launch.
constexpr int TS_NT = 256, TS_Q = 32, TS_TB = 64;
// acc[q][r] −= Σ_c M[r][c]·x[c][q] for r < m, c < mm, q < nq; M (TS_TB × TS_TB, ld TS_TB) and x in
// shared memory; thread → (row r, group of 8 RHS)
__device__ __forceinline__ void tile_gemv_sub(const cplx* __restrict__ Ms, const cplx* __restrict__ x,
                                              cplx* __restrict__ acc, int m, int mm, int nq) {
  for (int e = threadIdx.x; e < TS_TB * ((nq + 7) / 8); e += TS_NT) {
    const int r = e % TS_TB, qg = e / TS_TB;
    if (r >= m) continue;
    cplx sacc[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) sacc[w] = cmk(0.0, 0.0);
    for (int c = 0; c < mm; ++c) {
      const cplx a = Ms[r + c * TS_TB];
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc[w] = cfma(a, x[(qg * 8 + w) * TS_TB + c], sacc[w]);
    }
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int q = qg * 8 + w;
      if (q < nq) acc[q * TS_TB + r] = csub(acc[q * TS_TB + r], sacc[w]);
    }
  }
}
// M tile (rows o.., columns oo..) of the n × n column-major A into shared memory: every thread issues
// its 16 loads before using any (no dependent-latency chain)
__device__ __forceinline__ void load_tile(const cplx* __restrict__ A, int lda, int o, int m, int oo, int mm,
                                          cplx* __restrict__ Ms) {
  cplx v[TS_TB * TS_TB / TS_NT];
#pragma unroll
  for (int u = 0; u < TS_TB * TS_TB / TS_NT; ++u) {
    const int e = threadIdx.x + u * TS_NT, r = e % TS_TB, c = e / TS_TB;
    v[u] = (r < m && c < mm) ? __ldg(&A[(o + r) + (size_t)(oo + c) * lda]) : cmk(0.0, 0.0);
  }
#pragma unroll
  for (int u = 0; u < TS_TB * TS_TB / TS_NT; ++u) Ms[threadIdx.x + u * TS_NT] = v[u];
}

// Blocked triangular solve on Y (n × nq, ld ldy, nq ≤ TS_Q) with the LU in A: lower (unit L,
// forward) or upper (U, backward).  Blocks of TS_TB rows; a CTA takes the next block in dependency
// order from *ticket (every block it waits on is then already running), and for each earlier block:
// loads that off-diagonal tile into shared memory (independent of the chain, so it overlaps the
// wait), waits for the block's release flag, subtracts tile · rows; finally multiplies by its
// diagonal-block inverse, writes its rows and releases its flag.  flags[nblk], *ticket zero at launch.
__global__ void __launch_bounds__(TS_NT) k_lu_trsv(const cplx* __restrict__ A, int lda, int n,
                                                   const cplx* __restrict__ Dinv, cplx* Y, int ldy, int nq,
                                                   int upper, int* flags, int* ticket) {
  extern __shared__ __align__(16) unsigned char ts_sh[];
  cplx* acc = reinterpret_cast<cplx*>(ts_sh);  // [TS_Q][TS_TB]
  cplx* xb = acc + TS_Q * TS_TB;               // [TS_Q][TS_TB] rows of the block being subtracted
  cplx* Ms = xb + TS_Q * TS_TB;                // [TS_TB][TS_TB] tile
  __shared__ int tk;
  const int nblk = (n + TS_TB - 1) / TS_TB;
  if (threadIdx.x == 0) tk = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = tk;
  if (t >= nblk) return;
  const int b = upper ? nblk - 1 - t : t;
  const int o = b * TS_TB, m = min(TS_TB, n - o);
  for (int e = threadIdx.x; e < TS_Q * TS_TB; e += TS_NT) {
    const int r = e % TS_TB, q = e / TS_TB;
    acc[e] = (r < m && q < nq) ? Y[(o + r) + (size_t)q * ldy] : cmk(0.0, 0.0);
  }
  for (int u = 0; u < t; ++u) {  // dependencies in the order they complete
    const int bb = upper ? nblk - 1 - u : u;
    const int oo = bb * TS_TB, mm = min(TS_TB, n - oo);
    __syncthreads();  // previous tile consumed
    load_tile(A, lda, o, m, oo, mm, Ms);
    if (threadIdx.x == 0) {
      volatile int* f = flags + bb;
      while (*f == 0) {
      }
      __threadfence();
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TS_Q * TS_TB; e += TS_NT) {
      const int r = e % TS_TB, q = e / TS_TB;
      xb[e] = (r < mm && q < nq) ? __ldcg(&Y[(oo + r) + (size_t)q * ldy]) : cmk(0.0, 0.0);
    }
    __syncthreads();
    tile_gemv_sub(Ms, xb, acc, m, mm, nq);
  }
  // x = Dinv_b · acc  (as acc' = 0 − (−Dinv)·acc through the same routine: xb ← acc, acc ← 0)
  __syncthreads();
  {
    const cplx* D = Dinv + ((size_t)b * 2 + upper) * TS_TB * TS_TB;
    cplx v[TS_TB * TS_TB / TS_NT];
#pragma unroll
    for (int u2 = 0; u2 < TS_TB * TS_TB / TS_NT; ++u2) {
      const cplx d = D[threadIdx.x + u2 * TS_NT];
      v[u2] = cmk(-d.x, -d.y);
    }
#pragma unroll
    for (int u2 = 0; u2 < TS_TB * TS_TB / TS_NT; ++u2) Ms[threadIdx.x + u2 * TS_NT] = v[u2];
  }
  for (int e = threadIdx.x; e < TS_Q * TS_TB; e += TS_NT) {
    xb[e] = acc[e];
    acc[e] = cmk(0.0, 0.0);
  }
  __syncthreads();
  tile_gemv_sub(Ms, xb, acc, m, m, nq);
  __syncthreads();
  for (int e = threadIdx.x; e < TS_Q * TS_TB; e += TS_NT) {
    const int r = e % TS_TB, q = e / TS_TB;
    if (r < m && q < nq) Y[(o + r) + (size_t)q * ldy] = acc[e];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(flags + b, 1);
}

// Triangular products for the forward apply: Z = U·Y (upper) or Z = L·Y (unit lower), TS_TB-row
// blocks, no dependencies; tiles staged in shared memory (negated, so the same subtract routine
// accumulates +tile·x).  Y, Z: n × nq (ld ldy), nq ≤ TS_Q, Z ≠ Y.
__global__ void __launch_bounds__(TS_NT) k_lu_trmv(const cplx* __restrict__ A, int lda, int n,
                                                   const cplx* __restrict__ Y, cplx* __restrict__ Z, int ldy,
                                                   int nq, int upper) {
  extern __shared__ __align__(16) unsigned char tm_sh[];
  cplx* acc = reinterpret_cast<cplx*>(tm_sh);  // [TS_Q][TS_TB]
  cplx* xb = acc + TS_Q * TS_TB;               // [TS_Q][TS_TB]
  cplx* Ms = xb + TS_Q * TS_TB;                // [TS_TB][TS_TB]
  const int o = blockIdx.x * TS_TB, m = min(TS_TB, n - o);
  const int nblk = (n + TS_TB - 1) / TS_TB;
  for (int e = threadIdx.x; e < TS_Q * TS_TB; e += TS_NT) acc[e] = cmk(0.0, 0.0);
  const int bl = upper ? blockIdx.x : 0, bh = upper ? nblk - 1 : blockIdx.x;
  for (int bb = bl; bb <= bh; ++bb) {
    const int oo = bb * TS_TB, mm = min(TS_TB, n - oo);
    __syncthreads();
    load_tile(A, lda, o, m, oo, mm, Ms);
    for (int e = threadIdx.x; e < TS_Q * TS_TB; e += TS_NT) {
      const int r = e % TS_TB, q = e / TS_TB;
      xb[e] = (r < mm && q < nq) ? Y[(oo + r) + (size_t)q * ldy] : cmk(0.0, 0.0);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TS_TB * TS_TB; e += TS_NT) {  // triangle of the diagonal block; negate
      const int r = e % TS_TB, c = e / TS_TB;
      cplx v = Ms[e];
      if (bb == (int)blockIdx.x) {
        if (upper) v = c >= r ? v : cmk(0.0, 0.0);
        else v = c < r ? v : (c == r ? cmk(1.0, 0.0) : cmk(0.0, 0.0));
      }
      Ms[e] = cmk(-v.x, -v.y);
    }
    __syncthreads();
    tile_gemv_sub(Ms, xb, acc, m, mm, nq);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < TS_Q * TS_TB; e += TS_NT) {
    const int r = e % TS_TB, q = e / TS_TB;
    if (r < m && q < nq) Z[(o + r) + (size_t)q * ldy] = acc[e];
  }
}

template <int MC>
void launch_panel(cplx* A, int lda, int n, int* piv, int j0, int jb, int* status, cudaStream_t st) {
  static bool init = false;  // per process: the attribute is a property of the function
  if (!init) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_lu_panel<MC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(LU_CL, 1, 1);
  cfg.blockDim = dim3(LU_NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = LU_CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FMMLU_CUDA(cudaLaunchKernelEx(&cfg, k_lu_panel<MC>, A, lda, n, piv, j0, jb, status));
}

size_t swap_smem(int jb, int n) {
  return (size_t)jb * jb * sizeof(cplx) + (size_t)SW_C * 2 * jb * sizeof(cplx) + (2 * (size_t)jb + n) * sizeof(int) + 16;
}

}  // namespace

int root_lu_max_n() { return LU_CL * LU_RMAX; }

int root_lu_tb(int n) {
  // row-block height of the triangular solves: every block's CTA must be able to run at once is NOT
  // required (tickets), but fewer, taller blocks shorten the dependency chain
  (void)n;
  return 64;
}

void root_lu_factor(cplx* A, int n, int* piv, int* status, cplx* Dinv, cudaStream_t st, cudaStream_t sp,
                    const GemmFn& gemm) {
  const int lda = n;
  if (n > root_lu_max_n()) throw Error(-6, "root block larger than the register LU panel supports");
  static size_t sw_cur = 0;
  if (swap_smem(kRootNB, n) > sw_cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_lu_swap_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)swap_smem(kRootNB, n)));
    sw_cur = swap_smem(kRootNB, n);
  }
  // Lookahead: the trailing update of outer panel J is split into the next panel's columns (first) and
  // the rest; the next panel is then factored on a side stream while the rest of the update runs on st
  // (the panel kernels are latency-bound 16-CTA clusters, the update is a DMMA GEMM: they share the GPU).
  // sp: the side stream (sp == st: no lookahead)
  const bool lookahead = sp != st;
  cudaEvent_t ev_cols = nullptr, ev_panel = nullptr;
  if (lookahead) {
    FMMLU_CUDA(cudaEventCreateWithFlags(&ev_cols, cudaEventDisableTiming));
    FMMLU_CUDA(cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming));
    FMMLU_CUDA(cudaEventRecord(ev_cols, st));  // the block is built on st
  }
  try {
    for (int J0 = 0; J0 < n; J0 += kRootNB) {
      const int NB = std::min(kRootNB, n - J0);
      if (lookahead) FMMLU_CUDA(cudaStreamWaitEvent(sp, ev_cols, 0));  // this panel's columns are up to date
      for (int j0 = J0; j0 < J0 + NB; j0 += kRootIB) {
        const int jb = std::min(kRootIB, J0 + NB - j0);
        launch_panel<kRootIB>(A, lda, n, piv, j0, jb, status, sp);
        const int cw = NB;  // columns of J
        k_lu_swap_trsm<<<(cw + SW_C - 1) / SW_C, SW_NT, swap_smem(jb, n), sp>>>(A, lda, n, piv, j0, jb, J0, J0 + NB, j0,
                                                                              j0 + jb, j0 + jb);
        FMMLU_LAUNCH();
        const int m = n - (j0 + jb), nc = J0 + NB - (j0 + jb);
        if (m > 0 && nc > 0)
          gemm(sp, m, nc, jb, A + (j0 + jb) + (size_t)j0 * lda, lda, A + j0 + (size_t)(j0 + jb) * lda, lda,
               A + (j0 + jb) + (size_t)(j0 + jb) * lda, lda);
      }
      if (lookahead) {
        FMMLU_CUDA(cudaEventRecord(ev_panel, sp));
        FMMLU_CUDA(cudaStreamWaitEvent(st, ev_panel, 0));
      }
      if (n > NB) {
        k_lu_swap_trsm<<<(n + SW_C - 1) / SW_C, SW_NT, swap_smem(NB, n), st>>>(A, lda, n, piv, J0, NB, 0, n, J0, J0 + NB,
                                                                            J0 + NB);
        FMMLU_LAUNCH();
      }
      const int m = n - (J0 + NB);
      if (m > 0) {
        const cplx* Lp = A + (J0 + NB) + (size_t)J0 * lda;
        const int nn = lookahead ? std::min(kRootNB, m) : 0;  // the next panel's columns first
        if (nn > 0) {
          gemm(st, m, nn, NB, Lp, lda, A + J0 + (size_t)(J0 + NB) * lda, lda, A + (J0 + NB) + (size_t)(J0 + NB) * lda, lda);
          FMMLU_CUDA(cudaEventRecord(ev_cols, st));
        }
        if (m - nn > 0)
          gemm(st, m, m - nn, NB, Lp, lda, A + J0 + (size_t)(J0 + NB + nn) * lda, lda,
               A + (J0 + NB) + (size_t)(J0 + NB + nn) * lda, lda);
      }
    }
  } catch (...) {
    if (lookahead) {
      cudaStreamSynchronize(sp);
      cudaEventDestroy(ev_cols);
      cudaEventDestroy(ev_panel);
    }
    throw;
  }
  if (lookahead) {
    FMMLU_CUDA(cudaEventRecord(ev_panel, sp));
    FMMLU_CUDA(cudaStreamWaitEvent(st, ev_panel, 0));
    FMMLU_CUDA(cudaEventDestroy(ev_cols));
    FMMLU_CUDA(cudaEventDestroy(ev_panel));
  }
  const int TB = root_lu_tb(n), nblk = (n + TB - 1) / TB;
  const size_t smem = 2 * (size_t)TB * TB * sizeof(cplx);
  static size_t cur = 0;
  if (smem > 48 * 1024 && smem > cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_lu_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  k_lu_diag_inv<<<dim3(nblk, 2), 256, smem, st>>>(A, lda, n, TB, Dinv);
  FMMLU_LAUNCH();
}

int root_lu_launches(int n) {
  int nl = 0;
  for (int J0 = 0; J0 < n; J0 += kRootNB) {
    const int NB = std::min(kRootNB, n - J0);
    for (int j0 = J0; j0 < J0 + NB; j0 += kRootIB) nl += 3;
    nl += 2;
  }
  return nl + 1;
}

void root_lu_solve(const cplx* A, int n, const cplx* Dinv, cplx* Y, int ldy, int nrhs, int* flags, cudaStream_t st) {
  const int TB = root_lu_tb(n), nblk = (n + TB - 1) / TB;
  if (TB != TS_TB) throw Error(-6, "root solve block height mismatch");
  const size_t smem = (2 * (size_t)TS_Q * TS_TB + (size_t)TS_TB * TS_TB) * sizeof(cplx);
  static size_t cur = 0;
  if (smem > 48 * 1024 && smem > cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_lu_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  // flags: 2 × (nblk + 1) ints per RHS chunk (lower, upper): [flags | ticket]
  for (int q0 = 0; q0 < nrhs; q0 += TS_Q) {
    const int nq = std::min(TS_Q, nrhs - q0);
    FMMLU_CUDA(cudaMemsetAsync(flags, 0, 2 * (size_t)(nblk + 1) * sizeof(int), st));
    for (int upper = 0; upper < 2; ++upper) {
      int* f = flags + upper * (nblk + 1);
      k_lu_trsv<<<nblk, TS_NT, smem, st>>>(A, n, n, Dinv, Y + (size_t)q0 * ldy, ldy, nq, upper, f, f + nblk);
      FMMLU_LAUNCH();
    }
  }
}

void root_lu_mult(const cplx* A, int n, cplx* Y, cplx* Z, int ldy, int nrhs, cudaStream_t st) {
  const int TB = root_lu_tb(n), nblk = (n + TB - 1) / TB;
  const size_t smem = (2 * (size_t)TS_Q * TS_TB + (size_t)TS_TB * TS_TB) * sizeof(cplx);
  static size_t cur = 0;
  if (smem > 48 * 1024 && smem > cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_lu_trmv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  for (int q0 = 0; q0 < nrhs; q0 += TS_Q) {
    const int nq = std::min(TS_Q, nrhs - q0);
    k_lu_trmv<<<nblk, TS_NT, smem, st>>>(A, n, n, Y + (size_t)q0 * ldy, Z + (size_t)q0 * ldy, ldy, nq, 1);
    FMMLU_LAUNCH();
    k_lu_trmv<<<nblk, TS_NT, smem, st>>>(A, n, n, Z + (size_t)q0 * ldy, Y + (size_t)q0 * ldy, ldy, nq, 0);
    FMMLU_LAUNCH();
  }
}

}  // namespace fmmlu
