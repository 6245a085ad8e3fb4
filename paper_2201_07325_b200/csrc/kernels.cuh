// Task descriptors and launchers for the libfmmlu device kernels.
#pragma once
#include <functional>
#include "common.cuh"

#include <vector>

namespace fmmlu {

// Gather-or-generate one dense block of the current scaled matrix Ã.
// Entry (i, j): global indices gi = gidx[rows_off+i], gj = gidx[cols_off+j]; if the pair of
// their previous-level owners (slot[...]) has a stored block (tab[si*ns+sj] >= 0) the value is
// copied from it at (pos_i, pos_j) with leading dimension bld[si], else it is the pure kernel
// entry √w_i K √w_j (½ on the diagonal).  dst is column-major with ld = rows.
struct BuildTask {
  long long dst;           // complex offset of the block's (0,0) in the destination arena
  int ldd;                 // destination leading dimension (= block rows)
  int rows_off, cols_off;  // offsets into gidx/slot/pos for the block's rows / cols
  int i0, j0, ni, nj;      // the sub-tile of the block this task fills
  int ns;                  // slot table dimension
  int tab_off;             // offset into tab (ns*ns entries)
  int bld_off;             // offset into bld (ns entries, row-slot leading dims)
};

// Device-side description of one level's block store (CSR over owners).
struct LevelMeta {
  const int* actoff;     // no+1: prefix of active counts (rows of owner a = actoff[a+1]-actoff[a])
  const int* gidx;       // Σ act: global tree-order index of each active
  const int* slot;       // Σ act: slot of the active's previous-level owner in a's slot list (-1: none)
  const int* pos;        // Σ act: position in that previous-level owner's active list
  const int* nbptr;      // no+1: CSR row pointers of the block-pair set
  const int* nbidx;      // #pairs: partner owner
  const long long* poff; // #pairs: complex offset of the block in the level arena
  const int* slptr;      // no+1: CSR of the previous-level owners each owner is made of
  const int* sllist;
  // column side (separate incoming/outgoing IDs: an owner's active columns are
  // as many as its active rows but other DOFs); equal to gidx / slot / pos otherwise
  const int* gidxc;
  const int* slotc;
  const int* posc;
};
// Build every block of the level store: task = (pair, tile) with 64×64 tiles.  Each entry is the
// carried-over value when the previous level stored the owners' child pair, else the kernel
// entry √w_i K √w_j (½ on the diagonal).
void launch_build_level(const int2* d_tasks, int ntasks, const int* d_pair_a, const LevelMeta& cur,
                        const LevelMeta& prev, int has_prev, const cplx* src_arena, cplx* dst_arena, const Geo& g,
                        double k, cudaStream_t st);

// End of a level: compact the level store to the still-active rows / columns (see k_compact_level).
void launch_compact_level(int npairs, const int* pair_a, const LevelMeta& cur, const int* newactoff,
                          const long long* newpoff, const int* fposr, const int* fposc, const cplx* src, cplx* dst,
                          cudaStream_t st);

// Copy a (possibly index-mapped / transposed) block.
//   !trans: dst(i,j) = src(rm(i), cm(j));   trans: dst(i,j) = src(cm(j), rm(i))
// rm(i) = rmap ? rmap[i] : i (rmap_off < 0 means identity), same for cm.
struct CopyTask {
  long long src, dst;  // complex offsets into src / dst arenas
  int lds, ldd;
  int rows, cols;      // dst dims
  int trans;
  int rmap_off, cmap_off;
  int tri;             // 1: zero the strictly-lower part of dst (upper-triangular R copies)
  int ti, tj;          // tile origin within the original block (for the tri test)
};
// Mirror the upper triangle of Hermitian b×b matrices (ld b) into the lower one.
void launch_herm_mirror(cplx* const* d_ptrs, const int* d_dims, int nmats, int bmax, cudaStream_t st);
// Split copy tasks larger than 256×256 into 256×256 chunks (one CTA each).
void split_copy_tasks(std::vector<CopyTask>& v);
int copy_tiles(int rows, int cols);                  // tiles split_copy_tasks makes of one task
int emit_copy_tiles(const CopyTask& t, CopyTask* out);  // writes them, returns the count

// Proxy rows of M (§5.1.3; readings C3-C5): rows row0 .. row0+nγ-1 hold
// s_γ K(y_ℓ, x_j) √w_j (outgoing, combined field with the box normals), rows row0+nγ ..
// row0+2nγ-1 hold s_γ G(x_j, y_ℓ) √w_j (incoming single layer, transposed).
struct ProxyTask {
  long long dst;  // complex offset of M
  int ld, row0, b, idx_off, ngamma;
  double cx, cy, cz, rho, sg;
  int mode;       // 0: both row groups; 1: the outgoing rows only, 2: the incoming rows only (at row0; f3)
  int pad;
};

// Per-box ID on M (m × b, ld = m): CPQR with stopping rule |R_jj| ≤ eps·|R_00| (reading C9).
struct IdTask {
  cplx* Mp;       // the (m × b, ld m) matrix holding R' = [R11 R12] in rows 0..k-1
  int m, b;
  int out_off;    // offset into perm output (b ints)
  long long T;    // complex offset of T (k × (b-k)) in the T arena (capacity b*b)
};

// Elimination record of one box (offsets in the factor arena, complex units, and index arena).
struct BoxRec {
  long long T, Xi, Up, Lp;  // T: k×r, Xinv: r×r, Up = X_RR⁻¹X_{R(S∪N)}: r×(k+nN), Lp slot holds X_{(S∪N)R}: (k+nN)×r
  int k, r, nN;
  int idxS, idxR, idxN;     // offsets into the index arena (global tree-order indices)
  int tmp;                  // offset (in units of r·nrhs rows) of the box's solve scratch
};

// (box, chunk) work items of the split solve kernels
struct SolveItem {
  int rec;    // BoxRec index
  int c0;     // first row (upward, rows of Lp) or first column (downward, columns of Up)
};

// gidxc / slotc / posc: the column side of the frame (nullptr: same as the rows)
void launch_build(const BuildTask* d_tasks, int ntasks, const int* gidx, const int* slot,
                  const int* pos, const long long* tab, const int* bld, const cplx* src_arena,
                  cplx* dst_arena, const Geo& g, double k, cudaStream_t st, const int* gidxc = nullptr,
                  const int* slotc = nullptr, const int* posc = nullptr);
void launch_copy(const CopyTask* d_tasks, int ntasks, const int* maps, const cplx* src_arena,
                 cplx* dst_arena, cudaStream_t st);
void launch_proxy(const ProxyTask* d_tasks, int ntasks, const int* gidx, cplx* ws, const Geo& g,
                  double k, cudaStream_t st, int ngmax);
// One corrected-seminormal-equations refinement of T (Gram-path ID): T += R11⁻¹R11⁻ᴴ Z.
struct RefineTask {
  const cplx* R;  // R11 (k × k upper, ld ldr) from the pivoted Cholesky (R' layout over G)
  const cplx* Z;  // M_Sᴴ (M_R − M_S T)  (k × r, ld k)
  cplx* T;        // k × r, ld k, updated in place
  int ldr, k, r, kmax;
};
void launch_refine_T(const RefineTask* d_tasks, int ntasks, int kmax, int rmax, cudaStream_t st);
void launch_trsm_T(const IdTask* d_tasks, const int* d_k, int ntasks, const cplx* ws,
                   cplx* tarena, cudaStream_t st, int bmax);
// Blocked in-place Gauss-Jordan inverse (partial pivoting) of a batch of matrices.
struct GjTask {
  cplx* A;   // n × n, ld lda, inverted in place
  cplx* Am;  // blocked path: n × nb scratch (panel minus identity); register path: exchange scratch
  cplx* Y;   // nb × n scratch (rows J of the other columns)
  int* piv;  // n pivot rows
  int lda, n;
};
int gj_panel_width(int nmax);  // panel width nb whose n×nb panel fits shared memory
void launch_gj_panel(const GjTask* d_tasks, int ntasks, int j0, int nb, int* d_status, cudaStream_t st, int nmax);
void launch_gj_swap(const GjTask* d_tasks, int ntasks, int j0, int nb, cudaStream_t st, int nmax);
// cluster-distributed panel (rows over ≤ 16 CTAs) for blocks too tall for one CTA's smem
int gj_panel_cluster_size(int nmax, int nb);  // 0 = does not fit
void launch_gj_panel_cluster(const GjTask* d_tasks, int ntasks, int j0, int nb, int* d_status, cudaStream_t st,
                             int nmax);
// register-resident cluster panel (16 CTAs, L2 exchange): width for nmax (0 = not usable) and
// exchange scratch per task (complex elements) for panel width nb
int gj_panel_reg_width(int nmax);
long long gj_panel_reg_scratch(int nb);
void launch_gj_panel_reg(const GjTask* d_tasks, int ntasks, int j0, int nb, int* d_status, cplx* xs,
                         cudaStream_t st, int nmax);
void launch_gj_unscramble(const GjTask* d_tasks, int ntasks, cplx* scratch, const long long* d_soff, cudaStream_t st,
                          int nmax);
// Whole-matrix Gauss-Jordan inverse resident in (distributed) shared memory: one CTA, or a
// cluster of ≤ 16 CTAs holding the columns cyclically.  Returns false when nmax is too large
// (the caller uses the blocked panel path).
int gj_dsm_cluster_size(int nmax);  // 0 = does not fit
bool launch_gj_dsm(const GjTask* d_tasks, int ntasks, int* d_status, cudaStream_t st, int nmax);
// Householder QR (pivot = 0: TSQR round, writes triu(R) to out) or CPQR with the reading-C9
// stopping rule (pivot = 1: writes R' = [R11 R12], pivot columns first then the redundant ones
// in ascending index, over rows 0..k-1 of A, plus perm and k) on matrices resident in the
// distributed shared memory of a thread-block cluster of ≤ 16 CTAs.
struct ClusterQrTask {
  cplx* A;
  cplx* out;
  int lda, m, b, ldo;
  int out_off;  // perm output offset (pivot = 1)
  int pad;
};
int hqr_cluster_size(int m, int b);  // CTAs needed to hold m × b (0 = too large)
int hqr_max_rows(int b, int CL);     // largest m that fits a CL-CTA cluster with b columns
// m_of / b_of: host arrays with each task's (m, b) (they size the cluster and its shared memory)
void launch_hqr_cluster(const ClusterQrTask* d_tasks, int ntasks, int pivot, int* perm_out, int* k_out, double eps,
                        cudaStream_t st, const int* m_of, const int* b_of, double eps_rank = 0.0,
                        int* keps_out = nullptr);
// Pivoted Cholesky of G = MᴴM (b × b) in a cluster, same outputs as the pivoted launch above
// (R' over G with ld b).  false if b is too large for a 16-CTA cluster.
bool launch_pchol_cluster(const ClusterQrTask* d_tasks, int ntasks, int* perm_out, int* k_out, double eps,
                          cudaStream_t st, int bmax);
// Register-resident pivoted Cholesky (b ≤ 512; same outputs as launch_pchol_cluster).  xs: exchange
// scratch of pchol_reg_scratch(bmax) complex elements per task.  false if bmax is too large.
long long pchol_reg_scratch(int bmax);
// only_flagged: process only the tasks with k_out[task] < 0 (those launch_pchol_ll gave up on).
bool launch_pchol_reg(const ClusterQrTask* d_tasks, int ntasks, int* perm_out, int* k_out, double eps, cplx* xs,
                      cudaStream_t st, int bmax, int only_flagged = 0);
// Left-looking pivoted Cholesky, one CTA per box (b ≤ 512; same outputs).  Boxes whose rank passes
// max(rows of R held in shared memory, b/2) are left untouched with k_out = −1 for launch_pchol_reg
// (only_flagged).  task.out: b × b scratch.  false if bmax is too large.
// eps_rank / keps_out (separate IDs): the pivoting stops at eps (< eps_rank) and keps_out receives
// the rank at eps_rank; no_abort: never give up (b ≤ 1024 then).
bool launch_pchol_ll(const ClusterQrTask* d_tasks, int ntasks, int* perm_out, int* k_out, double eps,
                     cudaStream_t st, int bmax, double eps_rank = 0.0, int* keps_out = nullptr,
                     bool no_abort = false);
// Separate IDs: klow[2j], klow[2j+1] ← min(max(keps[2j], keps[2j+1]), klow[·]) (see k_sep_ranks).
void launch_sep_ranks(int* klow, const int* keps, int npairs, cudaStream_t st);
// Global-memory blocked pivoted Cholesky for boxes beyond the cluster capacity.
struct PcholState {
  int j;       // pivots taken so far
  int active;  // 0 once the ε stop rule fired (or all columns pivoted)
  double d0;   // largest initial diagonal (‖M_c‖² max)
};
struct PcholBig {
  cplx* G;     // b × b Gram matrix (ld b); receives R' at the end
  cplx* R;     // b × b: R rows by natural column
  cplx* Rp;    // nb × b: the current panel's R rows
  double* d;   // b: Schur-complement diagonal
  int* done;   // b
  int* piv;    // b
  PcholState* state;
  int b, out_off, kslot, pad;
};
void launch_pchol_big_panel(const PcholBig* d_tasks, int ntasks, int nb, double eps, cudaStream_t st, int bmax);
void launch_pchol_big_finish(const PcholBig* d_tasks, int ntasks, int* perm_out, int* k_out, cudaStream_t st,
                             int bmax);
// Split solve sweeps for one phase:
//   up:   [a] t = y_R − Tᵀy_S → tmp, y_R ← X_RR⁻¹ t   [b] y_{S∪N} −= X_{(S∪N)R} y_R (= Lp t; row chunks)
//   down: [a] acc = Up y_{S∪N} (column chunks, atomics)    [b] y_R −= acc, y_S −= T y_R
constexpr int kSolveChunk = 32;
void launch_solve_up2(const BoxRec* d_recs, int nrec, const SolveItem* d_items, int nitems, const cplx* fac,
                      const int* idx, cplx* y, int ldy, int nrhs, cplx* tmp, cudaStream_t st, int kmax, int rmax);
void launch_solve_down2(const BoxRec* d_recs, int nrec, const SolveItem* d_items, int nitems, const cplx* fac,
                        const int* idx, cplx* y, int ldy, int nrhs, cplx* tmp, cudaStream_t st, int rmax,
                        int kmax);
// forward factored apply: per-phase W, D and V sweeps (see kernels.cu)
void launch_apply_copyX(const BoxRec* d_recs, const BoxRec* d_recsX, int nrec, const cplx* fac, cplx* dst,
                        cudaStream_t st);
void launch_apply_w(const BoxRec* d_recs, int nrec, const SolveItem* d_items, int nitems, const cplx* fac,
                    const int* idx, cplx* y, int ldy, int nrhs, cplx* tmp, cudaStream_t st, int rmax, int kmax);
void launch_apply_d(const BoxRec* d_recsX, int nrec, const cplx* xs, const int* idx, cplx* y, int ldy, int nrhs,
                    cplx* tmp, cudaStream_t st, int rmax);
void launch_apply_v(const BoxRec* d_recs, int nrec, const SolveItem* d_items, int nitems, const cplx* fac,
                    const int* idx, cplx* y, int ldy, int nrhs, cplx* tmp, cudaStream_t st, int rmax);
// ---- device tree front end: checks + bounding box (per-block partials: 6 doubles per block),
// quantisation + Morton keys, tree-order geometry (SoA x,y,z,nx,ny,nz,√w) and sorted q
int tree_scan_blocks(long long n);
void launch_tree_scan(const double* P, const double* N, const double* W, long long n, double* part, int* bad,
                      cudaStream_t st);
void launch_tree_keys(const double* P, long long n, const double lo[3], double side, unsigned long long* key, int* idx,
                      int* q, cudaStream_t st);
void launch_tree_gather(const double* P, const double* N, const double* W, long long n, const int* perm, const int* q,
                        double* G, long long* perm64, int* qs, cudaStream_t st);
// ---- multi-RHS sweeps on DMMA GEMMs: per-box dense blocks gathered from /
// scattered to the tree-order RHS y (ld ldy) around batched GEMMs.
struct SweepWs {   // complex offsets into the phase workspace, per box
  long long ysn;   // (k+nN) × Q: rows [S | N]
  long long yr;    // r × Q
  long long z;     // r × Q   (up: X_RR⁻¹ t)
  long long dsn;   // (k+nN) × Q (up: Lp t; down: T y_R in its first k rows)
};
// mode 0: YSN ← y[S∪N], YR ← y[R];  1: up scatter y[R] = Z, y[S∪N] −= DSN;  2: down scatter
// y[R] = YR, y[S] −= DSN[0:k].  grid (nrec, ceil(Q / qb)).
void launch_sweep_move(const BoxRec* d_recs, const SweepWs* d_ws, int nrec, const int* idx, cplx* y, int ldy,
                       int Q, cplx* ws, int mode, cudaStream_t st);
// y[rows[i], q] ↔ Y0[i + q n0] (dir 0: gather, 1: scatter)
void launch_rows_move(const int* rows, int n0, cplx* y, int ldy, cplx* Y0, int Q, int dir, cudaStream_t st);
// y[i + a·ldy] = −e^{ik x_i·d_a} √w_i (tree order, scaled: the solve's input W^{½}b), d_a = (cos φ_a, sin φ_a, 0)
void launch_plane_wave(Geo g, int n, double k, const double* phis, int Q, cplx* y, int ldy, cudaStream_t st);
// R[a] += (−ik/4π) Σ_i √w_i (1 − n_i·d_a) e^{ik x_i·d_a} y[i + a·ldy]   (y = W^{½}σ in tree order)
void launch_rcs_reduce(Geo g, int n, double k, const double* phis, int Q, const cplx* y, int ldy, cplx* R,
                       cudaStream_t st);
// y[rows] = Xinv (n0×n0) · y[rows] for the root block
void launch_root_apply(const cplx* Xinv, int n0, const int* d_rows, cplx* y, int ldy, int nrhs,
                       cplx* tmp, cudaStream_t st);
// elementwise helpers (caller order <-> tree order, √w scaling)
void launch_permute_in(const cplx* src, int ld_src, cplx* dst, int n, int nrhs,
                       const long long* perm, const double* sw, int mode, cudaStream_t st);
void launch_permute_out(const cplx* src, cplx* dst, int ld_dst, int n, int nrhs,
                        const long long* perm, const double* sw, int mode, cudaStream_t st);
// brute-force y = A x (unscaled, tree order; w = sw²)
void launch_matvec(const Geo& g, double k, int n, const cplx* x, cplx* y, int nrhs,
                   cudaStream_t st);
double probe_fp64(int kind);
// cfg4: row-major per-box geometry → SoA (x|y|z|nx|ny|nz|√w), box i at [i·(b+nnear), (i+1)·(b+nnear))
void launch_box_geo(const double* pts, const double* nrm, const double* npts, const double* nnrm, int nbox, int b,
                    int nnear, double sw, double* out, cudaStream_t st);

// ---- root block: blocked right-looking LU with partial pivoting, rootlu.cu
constexpr int kRootNB = 64;  // outer panel (trailing-update GEMM depth)
constexpr int kRootIB = 16;  // inner register panel width
// C −= A·B (m×n, k) on the library's DMMA GEMM; supplied by the host orchestration
using GemmFn = std::function<void(cudaStream_t s, int m, int n, int k, const cplx* A, int lda, const cplx* B, int ldb,
                                  cplx* C, int ldc)>;
int root_lu_max_n();
int root_lu_tb(int n);  // row-block height of the blocked triangular solves / Dinv blocks
// In place P·A = L·U of the n × n column-major A (ld n); piv[j] = row interchanged with j at step j;
// Dinv (2·ceil(n/TB)·TB² complex): inverses of L's and U's TB × TB diagonal blocks; *status = 1 on an
// exactly zero pivot column.  sp: side stream for the lookahead (the next outer panel is factored on it
// while the rest of the trailing update runs on st); sp == st: none.  gemm(s, ...) runs C −= A·B on s.
void root_lu_factor(cplx* A, int n, int* piv, int* status, cplx* Dinv, cudaStream_t st, cudaStream_t sp,
                    const GemmFn& gemm);
int root_lu_launches(int n);
// Y (n × nrhs, ld ldy, rows already permuted by P) ← U⁻¹ L⁻¹ Y.  flags: 2·(ceil(n/TB)+1) ints scratch.
void root_lu_solve(const cplx* A, int n, const cplx* Dinv, cplx* Y, int ldy, int nrhs, int* flags, cudaStream_t st);
// Y ← L·U·Y (Z: n × nrhs scratch, ld ldy); the caller applies Pᵀ when scattering.
void root_lu_mult(const cplx* A, int n, cplx* Y, cplx* Z, int ldy, int nrhs, cudaStream_t st);

}  // namespace fmmlu
