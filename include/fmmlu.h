/*
 * fmmlu.h — C ABI of the B200-native FMM-LU hot path (libfmmlu.so).
 *
 * The library factorizes and solves the dense combined-field Helmholtz
 * Nyström system of PAPER.md Eq. disc1 (L443-450) with the BASELINE.json
 * conventions:
 *
 *     A = ½ I + (D − i k S) W,   K(x,y) = n(y)·∇_y G(x,y) − i k G(x,y),
 *     G(x,y) = e^{ik|x−y|}/(4π|x−y|),   K(x_i,x_i) := 0,   W = diag(w)
 *
 * (PAPER.md L408-421 Eqs. greenfunhelm/comb_ref, L2033-2038 Eq. num-inteq),
 * by recursive strong skeletonization (RS-S) over a level-restricted adaptive
 * octree (§4) with proxy-surface compression and the
 * simultaneous incoming/outgoing interpolative decomposition of PAPER.md §5.1
 * (L1373-1914).  Internally the √w-scaled matrix Ã = W^{½} A W^{−½} is
 * factorized (PAPER.md Eq. disc3); results are in A's variables.
 *
 * Memory: every array argument may be a HOST pointer or a CUDA DEVICE pointer
 * on the current device (detected with cudaPointerGetAttributes).  Host
 * arguments are copied in (and, for fmmlu_solve, back out) inside the call.
 * Complex numbers are interleaved (re, im) doubles (= C99 double complex =
 * cuDoubleComplex = torch.complex128).  The caller keeps ownership of all
 * argument buffers; the handle owns all internal device memory.
 *
 * Streams: all device work is issued on the handle's stream (default: a
 * non-blocking stream the handle creates; see fmmlu_set_stream).  fmmlu_tree,
 * fmmlu_factor and fmmlu_solve return after their work is complete.
 * Ordering precondition for DEVICE arguments: the library orders its work after
 * everything already queued on the legacy default stream, and (after
 * fmmlu_set_stream) on the given stream; a device buffer written on any OTHER
 * stream must be complete (that stream synchronised) before the call.  The
 * Python binding synchronises torch's current stream for CUDA tensors.
 *
 * Device memory: handles allocate from a private stream-ordered pool of the
 * library (never the device's default pool).  Large blocks and the per-device
 * factorization workspace are kept across handles for reuse;
 * fmmlu_release_cache() returns them to the driver.
 *
 * Errors: every function returns 0 on success or a negative FMMLU_E* code;
 * fmmlu_last_error() gives a human-readable message for the calling thread's
 * last failure.  No function aborts the process.
 *
 * Concurrency: a handle is single-threaded (one call at a time).  There is no
 * CPU fallback: the compute path runs only on the GPU and fails with
 * FMMLU_ECUDA if no usable sm_100 device is present.
 */
#ifndef FMMLU_H
#define FMMLU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMMLU_OK 0
#define FMMLU_EINVAL (-1)    /* bad argument (see each function)                         */
#define FMMLU_EDEPTH (-2)    /* tree deeper than 20 levels (duplicate points) */
#define FMMLU_ESINGULAR (-3) /* exactly singular pivot block X_RR or root block          */
#define FMMLU_ENOMEM (-4)    /* device or host allocation failed                         */
#define FMMLU_ESTATE (-5)    /* call order violated (e.g. solve before factor)           */
#define FMMLU_ENOTIMPL (-6)  /* stage not built                                          */
#define FMMLU_ECUDA (-7)     /* CUDA runtime / launch error                              */

typedef struct fmmlu_handle fmmlu_handle;

typedef struct fmmlu_stats_t {
  int64_t n;              /* number of unknowns                                   */
  int32_t nlevels;        /* octree levels (0 .. nlevels-1) after 2:1 balancing  */
  int32_t nboxes;         /* boxes in the tree                                    */
  int32_t nleaves;        /* leaf boxes                                           */
  int32_t n_eliminated;   /* boxes skeletonized (with |R| > 0)                    */
  int64_t n0;             /* size of the dense root block B_t */
  int32_t max_rank;       /* largest |S| over skeletonized boxes                  */
  int32_t max_b;          /* largest number of actives in a skeletonized box      */
  int64_t factor_bytes;   /* device bytes held by the factor store                */
  int64_t peak_bytes;     /* device high-water mark of the handle                 */
  double t_tree_ms;       /* last fmmlu_tree wall time                            */
  double t_factor_ms;     /* last fmmlu_factor wall time                          */
  double t_solve_ms;      /* last fmmlu_solve wall time                           */
  double t_root_ms;       /* root LU part of the last factor                      */
  double t_levels_ms[24]; /* per-level part of the last factor (index = level)    */
  int32_t n_singular_warn;/* near-singular pivot warnings                         */
  int32_t ranks_sum[24];  /* Σ|S| per level                                       */
  int32_t boxes[24];      /* skeletonized boxes per level                         */
  int64_t n_launches;     /* kernels launched by the last tree + factor + solve   */
  /* Per kernel class (FMMLU_K_* below), accumulated over the last factor and the
   * last solve: device time from CUDA events recorded on the launch stream, and the
   * ALGORITHMIC real flops / bytes of the launches in that class.                 */
  double class_ms[16];
  double class_flops[16];
  double class_bytes[16];
  int64_t class_launches[16];
  double t_sync_wait_ms;  /* part of t_factor_ms the host spent blocked on the stream */
} fmmlu_stats_t;

/* kernel classes for fmmlu_stats_t.class_* */
#define FMMLU_K_BUILD 0   /* level block store: kernel generation + carry-over      */
#define FMMLU_K_GATHER 1  /* M / W gathers, proxy rows                              */
#define FMMLU_K_QR 2      /* ID: Householder QR of M                                */
#define FMMLU_K_CPQR 3    /* ID: column-pivoted QR + T = R11^-1 R12                 */
#define FMMLU_K_EF 4      /* E/F transforms (GEMM)                                  */
#define FMMLU_K_INV 5     /* X_RR^-1 (Gauss-Jordan)                                 */
#define FMMLU_K_PANEL 6   /* Up = X_RR^-1 X_R(S+N) panel (GEMM)                     */
#define FMMLU_K_SCHUR 7   /* Schur-complement GEMM + scatter-add                    */
#define FMMLU_K_ROOT 8    /* root block build + inverse                             */
#define FMMLU_K_SOLVE 9   /* solve sweeps + root apply                              */
#define FMMLU_K_APPLY 10  /* forward apply sweeps (+ one-time re-inversion of D)    */
#define FMMLU_K_NCLASS 11

/* Build the adaptive level-restricted octree over the n points
 * (readings C14, C6-C8 of SURVEY.md §8(c)).
 *   points  : n×3 row-major (x0,y0,z0,x1,...) fp64, host or device
 *   normals : n×3 row-major unit outward normals n(x_i)
 *   weights : n smooth quadrature weights w_i > 0
 *   n       : ≥ 1;  leaf_max : s ≥ 1 (split a box while it holds more than s points)
 *   out     : receives a new handle (set to NULL on failure)
 * Errors: EINVAL (n < 1, leaf_max < 1, NULL pointer, w ≤ 0 or non-finite,
 * |‖n_i‖ − 1| > 1e-10), EDEPTH, ENOMEM, ECUDA. */
int fmmlu_tree(const double* points, const double* normals, const double* weights,
               int64_t n, int leaf_max, fmmlu_handle** out);

/* Factorize A (wavenumber k, η = k) by RS-S at ID tolerance eps
 * (ID per L606-638 with the stopping rule of reading C9;
 * proxy surface per readings C4/C5).  Replaces any previous factorization.
 * Errors: EINVAL (k ≤ 0 or non-finite, eps ∉ (0,1)), ESINGULAR, ENOMEM, ECUDA. */
int fmmlu_factor(fmmlu_handle* h, double k, double eps);

/* Solve A x = b in place for nrhs right-hand sides (PAPER.md L920-924:
 * A⁻¹ ≈ W₁⁻¹⋯W_M⁻¹ P_t D⁻¹ P_tᵀ V_M⁻¹⋯V₁⁻¹, sign-toggled factors L833-858).
 *   rhs  : n×nrhs column-major complex128 (host or device); in: b, out: x
 *   nrhs : ≥ 1
 * The handle keeps n×nrhs complex work buffers between calls for nrhs < 32 (repeated solves with the
 * same nrhs replay one captured CUDA graph); they are released by fmmlu_destroy.
 * Errors: EINVAL (NULL rhs, nrhs < 1), ESTATE (no factorization), ENOMEM, ECUDA. */
int fmmlu_solve(fmmlu_handle* h, void* rhs, int nrhs);

/* Forward factored apply, in place: x ← Â x with the stored factors
 * Â = V₁⋯V_M P_t D P_tᵀ W_M⋯W₁ ≈ A  (V = P E⁻¹ L⁻¹, W = U⁻¹ F⁻¹ Pᵀ
 * with sign-toggled inverses L851-853; D = diag(X_{R_jR_j}, A_{B_tB_t})).  Exactly
 * inverse to fmmlu_solve up to rounding, and within the factorization's ε of A x.
 * The first call after a factorization re-inverts the stored X_RR⁻¹ / X_t⁻¹
 * blocks (reading R3) into a cache of the same size, held until the next factor.
 *   x    : n×nrhs column-major complex128 (host or device), caller ordering
 *   nrhs : ≥ 1
 * Errors: EINVAL (NULL x, nrhs < 1), ESTATE (no factorization), ESINGULAR, ENOMEM, ECUDA. */
int fmmlu_apply(fmmlu_handle* h, void* x, int nrhs);

/* Azimuthal monostatic sonar cross section of the sound-soft scatterer (§6.3,
 * L2755-2794): for each φ_a, d = (cos φ_a, sin φ_a, 0), solve A σ = −e^{ik x·d}
 * with the stored factors (k = the factorization's wavenumber) and return
 *   R(φ_a) = (−ik/4π) Σ_j w_j (1 − n_j·d) e^{+ik x_j·d} σ_j     (reading R8 of DESIGN.md).
 * Right-hand sides are generated on the device; ≥ 32 angles run the sweeps as batched DMMA GEMMs.
 *   phis : nphi azimuths (radians), host or device;  R : nphi complex128 out, host or device
 * Errors: EINVAL (NULL, nphi < 1), ESTATE (no factorization), ENOMEM, ECUDA. */
int fmmlu_monostatic_rcs(fmmlu_handle* h, const double* phis, int nphi, void* R);

/* Apply the (unfactored) matrix: y = A x by brute-force O(n²) summation on the
 * GPU (test/measurement infrastructure for residuals; reading C17).
 *   x, y : n×nrhs column-major complex128 (host or device; y may not alias x)
 * Errors: EINVAL, ESTATE (no tree), ECUDA. */
int fmmlu_matvec(fmmlu_handle* h, double k, const void* x, void* y, int nrhs);

/* Return the library's cached device memory (per-device factorization workspace,
 * large-block cache, idle pool reservation) to the driver, on every device.  Call
 * when no handle is in the middle of a call; live handles keep their factors.
 * Errors: ECUDA. */
int fmmlu_release_cache(void);

/* Release the handle and all device memory it owns.  NULL is a no-op. */
int fmmlu_destroy(fmmlu_handle* h);

/* Message for the calling thread's most recent failure ("" if none). */
const char* fmmlu_last_error(void);

/* Statistics of the handle's tree / last factor / last solve. */
int fmmlu_stats(const fmmlu_handle* h, fmmlu_stats_t* out);

/* Issue subsequent work on cuda_stream (a cudaStream_t; NULL = the handle's
 * own stream).  The caller keeps ownership of the stream. */
int fmmlu_set_stream(fmmlu_handle* h, void* cuda_stream);

/* Tuning parameters (apply to the next fmmlu_factor):
 *   "id_mode"   0 = auto (Gram path where eps^2 >= 4*b_max*u, Householder below; default),
 *               1 = Householder TSQR + column-pivoted QR on the ID matrix,
 *               2 = Gram matrix + pivoted Cholesky (same pivots/rank/T as CPQR in exact
 *                   arithmetic; accurate while eps^2 >> unit roundoff)
 *               3 = as 2 but always with the global-memory blocked pivoted Cholesky
 *                   (the path used automatically for boxes beyond the cluster capacity)
 *   "id_refine" 0..3 corrected-seminormal-equations steps on the Gram-path T of fmmlu_boxes
 *               (each contracts the T error by ~u*cond(M_S)^2, to the u*cond(M_S) of a
 *               Householder ID; R4); fmmlu_boxes uses 2
 *   "pchol_mode" Gram-path pivoted Cholesky: 0 = register-resident kernel (b <= 512; default),
 *               1 = shared-memory cluster kernel
 *   "gj_mode"   X_RR inverse (Gauss-Jordan, partial pivoting): 0 = auto (whole matrix resident
 *               in one CTA's or one <=16-CTA cluster's shared memory when it fits, blocked
 *               panel path otherwise; default), 1 = blocked panel path always
 *   "proxy_rho" proxy-sphere radius / box side, in (sqrt(3)/2, 5/2) (reading C5; default 2.0)
 *   "separate_id" 0 = one simultaneous ID of [A_QB; A_BQ^T; proxy rows] per box (default),
 *               1 = separate incoming / outgoing interpolation matrices (PAPER.md L726-732,
 *               L1098-1108, L1909-1914; R12): a column ID of
 *               M_c = [A_QB; outgoing proxy rows] gives (S_c, T_c) and a row ID of
 *               M_r = [A_BQ^T; incoming proxy rows] gives (S_r, T_r); both sides keep
 *               k = max(k_c, k_r) skeletons so that X_RR stays square; a box then keeps
 *               different active rows and columns, and fmmlu_solve / fmmlu_apply carry the
 *               vector from the equation side to the unknown side between the sweeps
 *   "deterministic" 0 / 1 (R9)
 * Errors: EINVAL (unknown name or value out of range). */
int fmmlu_set_param(fmmlu_handle* h, const char* name, double value);

/* The octree's boxes (built on the device): level-major, Morton order within a
 * level.  Call with all arrays NULL to get the count in *nboxes; otherwise *nboxes is the capacity
 * on entry and the count on return.  level[b], coord[3b..3b+2] (cell coordinates at that level),
 * start[b]/end[b] (point range in tree order; fmmlu_tree_perm maps tree positions to caller
 * indices).  Host arrays.  Errors: EINVAL (NULL nboxes, capacity too small). */
int fmmlu_tree_boxes(const fmmlu_handle* h, int32_t* nboxes, int32_t* level, int32_t* coord, int32_t* start,
                     int32_t* end);

/* The owner lists of one level (2 <= level < nlevels), as built on the device from the finished
 * tree (PAPER.md L563-565 neighbours, L1263-1267 far-field neighbours; readings C6,
 * C7): the owners at that level are its boxes followed by the leaves of the coarser levels (box
 * ids as in fmmlu_tree_boxes); for the j-th level box, N = owners[nidx[nptr[j] .. nptr[j+1])]
 * (separation <= 1 in level cells) and Q = owners[qidx[qptr[j] .. qptr[j+1])] (separation 2), both
 * ascending in the local owner index.  counts[0..3] receive (#level boxes, #owners, |nidx|, |qidx|);
 * call with owners == NULL to get only the counts.  Host arrays: owners[#owners],
 * nptr / qptr [#level boxes + 1], nidx, qidx.  Colour of a level box = 4 (cx & 1) + 2 (cy & 1) +
 * (cz & 1) (reading C8).  Errors: EINVAL (NULL argument, level out of range). */
int fmmlu_level_lists(fmmlu_handle* h, int level, int32_t* counts, int32_t* owners, int32_t* nptr, int32_t* nidx,
                      int32_t* qptr, int32_t* qidx);

/* Tree order: perm[i] = caller index of the i-th point in tree (Morton) order.
 * perm: int64[n] host buffer. */
int fmmlu_tree_perm(const fmmlu_handle* h, int64_t* perm);

/* Batched in-place inverse of the X_RR blocks' kind (the elimination applies
 * X_RR^-1; reading R3: explicit inverse by Gauss-Jordan with partial pivoting), exposed for
 * kernel-level tests and timing.  A: DEVICE pointer to `count` n x n complex128 matrices,
 * column-major, contiguous (matrix c at A + c*n*n*16 bytes), inverted in place on the
 * handle's stream with the handle's "gj_mode".  ms (optional, may be NULL): device time of the
 * inversion (CUDA events).  Synchronises the stream.
 * Errors: EINVAL (NULL, host pointer, n < 1, count < 1), ESINGULAR (an exactly zero pivot). */
int fmmlu_inverse_batch(fmmlu_handle* h, void* A, int n, int count, double* ms);

/* Config-4 workload (BASELINE.json configs[3], readings C21/C22): ID and
 * elimination of nbox INDEPENDENT boxes (one level, nothing modified yet, Q = ∅).
 *   pts, nrm   : nbox × b × 3 doubles (row-major xyz per point): box points, unit normals
 *   npts, nnrm : nbox × nnear × 3: the near set N of each box (Schur-update targets, C22)
 *   w          : uniform quadrature weight; k: wavenumber; eps: ID tolerance (0,1)
 *   n_gamma, rho: proxy points (Fibonacci directions, R2) on the sphere of radius rho about
 *               the origin (every box is centred at 0); ID rows = 2 n_gamma proxy rows (C21)
 * Per box: M = [s_γ K(y_ℓ,x_j)√w ; s_γ G(x_j,y_ℓ)√w], ID (L606-638,
 * C9), E/F transforms, X_RR^-1, panels, and Δ = −X_{(S∪N)R} X_RR^-1 X_{R(S∪N)} (L753-825).
 * Outputs (host or device pointers):
 *   ranks  int32[nbox]: k of each box
 *   perm   int32[nbox × b] or NULL: skeleton columns first (pivot order), then the redundant
 *          ones ascending
 *   keep[nkeep], delta: for box keep[j], Δ ((k+nnear) × (k+nnear), column-major, frame
 *          [S in pivot order | N]) is written at delta + j·(b+nnear)² complex128 elements
 *   timing double[3] or NULL: device ms of the whole batch, model GFLOP (SURVEY §8(d) cost
 *          model with the measured ranks), boxes per wave.
 * Errors: EINVAL, ENOMEM, ESINGULAR (exactly singular X_RR), ECUDA. */
int fmmlu_boxes(const double* pts, const double* nrm, const double* npts, const double* nnrm, int nbox, int b,
                int nnear, double w, double k, double eps, int n_gamma, double rho, int* ranks, int* perm,
                int nkeep, const int* keep, void* delta, double* timing);

/* Measure FP64 peak on this device: DFMA (kind=0) or DMMA m8n8k4 (kind=1)
 * throughput in TFLOP/s (roofline denominator; not part of the method). */
int fmmlu_probe_fp64(int kind, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* FMMLU_H */
