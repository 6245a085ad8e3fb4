// libfmmlu device kernels (sm_100a): block builder (kernel generation + Schur
// state carry-over), gathers, proxy rows, CPQR ID, T solve, Gauss-Jordan
// inverses, solve sweeps, brute-force matvec, FP64 probes.
#include <cooperative_groups.h>

#include <cfloat>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fmmlu {

namespace {

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

template <int NT>
__device__ void block_argmax(double& v, int& idx, double* sv, int* si) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    argmax_merge(v, idx, v2, i2);
  }
  if (lane == 0) {
    sv[w] = v;
    si[w] = idx;
  }
  __syncthreads();
  if (w == 0) {
    v = lane < NT / 32 ? sv[lane] : -1.0;
    idx = lane < NT / 32 ? si[lane] : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      argmax_merge(v, idx, v2, i2);
    }
    if (lane == 0) {
      sv[0] = v;
      si[0] = idx;
    }
  }
  __syncthreads();
  v = sv[0];
  idx = si[0];
  __syncthreads();
}

template <int NT>
__device__ double block_sum(double v, double* sv) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sv[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < NT / 32 ? sv[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sv[0] = v;
  }
  __syncthreads();
  v = sv[0];
  __syncthreads();
  return v;
}

__device__ __forceinline__ cplx warp_csum(cplx v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ block builder
__global__ void k_build(const BuildTask* __restrict__ tasks, const int* __restrict__ gidx,
                        const int* __restrict__ slot, const int* __restrict__ pos,
                        const long long* __restrict__ tab, const int* __restrict__ bld,
                        const cplx* __restrict__ src, cplx* __restrict__ dst, Geo g, double k) {
  const BuildTask t = tasks[blockIdx.x];
  const int n = t.ni * t.nj;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int i = t.i0 + e % t.ni, j = t.j0 + e / t.ni;
    const int ri = t.rows_off + i, cj = t.cols_off + j;
    const int si = slot[ri], sj = slot[cj];
    cplx v;
    long long off = -1;
    if (si >= 0 && sj >= 0) off = tab[t.tab_off + si * t.ns + sj];
    if (off >= 0) {
      v = src[off + pos[ri] + (size_t)pos[cj] * bld[t.bld_off + si]];
    } else {
      v = entry_scaled(g, k, gidx[ri], gidx[cj]);
    }
    dst[t.dst + i + (size_t)j * t.ldd] = v;
  }
}

// ------------------------------------------------------------------ copies
__global__ void k_copy(const CopyTask* __restrict__ tasks, const int* __restrict__ maps,
                       const cplx* __restrict__ src, cplx* __restrict__ dst) {
  const CopyTask t = tasks[blockIdx.x];
  const int n = t.rows * t.cols;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int i = e % t.rows, j = e / t.rows;
    const int ri = t.rmap_off >= 0 ? maps[t.rmap_off + i] : i;
    const int cj = t.cmap_off >= 0 ? maps[t.cmap_off + j] : j;
    cplx v = t.trans ? src[t.src + cj + (size_t)ri * t.lds] : src[t.src + ri + (size_t)cj * t.lds];
    if (t.tri && i > j) v = cmk(0.0, 0.0);
    dst[t.dst + i + (size_t)j * t.ldd] = v;
  }
}

// ------------------------------------------------------------------ proxy rows
__global__ void k_proxy(const ProxyTask* __restrict__ tasks, const int* __restrict__ gidx,
                        cplx* __restrict__ ws, Geo g, double k) {
  const ProxyTask t = tasks[blockIdx.x];
  const double ga = M_PI * (3.0 - sqrt(5.0));
  const int n = t.ngamma * t.b;
  for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < n; e += blockDim.x * gridDim.y) {
    const int l = e % t.ngamma, j = e / t.ngamma;
    // Fibonacci direction u_l (reading C5)
    const double zl = 1.0 - (2.0 * l + 1.0) / t.ngamma;
    const double phi = l * ga;
    const double s = sqrt(fmax(0.0, 1.0 - zl * zl));
    double sp, cp;
    sincos(phi, &sp, &cp);
    const double yx = t.cx + t.rho * s * cp, yy = t.cy + t.rho * s * sp, yz = t.cz + t.rho * zl;
    const int gj = gidx[t.idx_off + j];
    const double xx = g.x[gj], xy = g.y[gj], xz = g.z[gj];
    const double scl = t.sg * g.sw[gj];
    // outgoing: K(y_l, x_j) with source normal n(x_j)
    cplx Ko = kernel_K(k, yx - xx, yy - xy, yz - xz, g.nx[gj], g.ny[gj], g.nz[gj]);
    // incoming: G(x_j, y_l)
    cplx Gi = kernel_G(k, xx - yx, xy - yy, xz - yz);
    ws[t.dst + (t.row0 + l) + (size_t)j * t.ld] = cscale(Ko, scl);
    ws[t.dst + (t.row0 + t.ngamma + l) + (size_t)j * t.ld] = cscale(Gi, scl);
  }
}

// ------------------------------------------------------------------ blocked Householder QR panel
// Hermitian reflectors H = I − τ v vᴴ (τ real, v_0 = 1) with H x = β e1, β = −(α/|α|)‖x‖.
constexpr int QP_NT = 512;
constexpr int QP_NBMAX = 16;

__global__ void __launch_bounds__(QP_NT) k_qr_panel(const QrChunk* __restrict__ chunks, int j0, int NB) {
  extern __shared__ double shm[];
  __shared__ double red_v[32];
  __shared__ cplx sred[QP_NT / 32][QP_NBMAX];
  __shared__ cplx dots[QP_NBMAX];
  __shared__ double tau[QP_NBMAX];
  __shared__ cplx G[QP_NBMAX][QP_NBMAX];
  __shared__ cplx Tm[QP_NBMAX][QP_NBMAX];
  const QrChunk c = chunks[blockIdx.x];
  const int kmax = min(c.h, c.b);
  if (j0 >= kmax) return;
  const int jb = min(NB, kmax - j0);
  const int hr = c.h - j0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  cplx* P = reinterpret_cast<cplx*>(shm);  // hr × jb, ld hr
  cplx* A = c.A;
  for (int e = tid; e < hr * jb; e += QP_NT) {
    const int i = e % hr, jj = e / hr;
    P[e] = A[(j0 + i) + (size_t)(j0 + jj) * c.lda];
  }
  __syncthreads();
  for (int jj = 0; jj < jb; ++jj) {
    double xs = 0.0;
    for (int i = jj + 1 + tid; i < hr; i += QP_NT) xs += cabs2(P[i + jj * hr]);
    const double xn2 = block_sum<QP_NT>(xs, red_v);
    const cplx alpha = P[jj + jj * hr];
    const double aa = sqrt(cabs2(alpha));
    const double nrm = sqrt(aa * aa + xn2);
    __syncthreads();
    if (nrm == 0.0) {  // zero column: identity reflector
      if (tid == 0) tau[jj] = 0.0;
      __syncthreads();
      continue;
    }
    const cplx beta = aa > 0.0 ? cmk(-alpha.x / aa * nrm, -alpha.y / aa * nrm) : cmk(-nrm, 0.0);
    const cplx u0 = csub(alpha, beta);
    const double u02 = cabs2(u0);
    const cplx inv_u0 = cmk(u0.x / u02, -u0.y / u02);
    for (int i = jj + 1 + tid; i < hr; i += QP_NT) P[i + jj * hr] = cmul(P[i + jj * hr], inv_u0);
    if (tid == 0) {
      tau[jj] = 2.0 * u02 / (u02 + xn2);
      P[jj + jj * hr] = beta;
    }
    __syncthreads();
    const int nrest = jb - jj - 1;
    if (nrest > 0) {
      // d_c = vᴴ P[jj:, c] for the remaining panel columns (v_jj = 1)
      cplx d[QP_NBMAX];
#pragma unroll
      for (int q = 0; q < QP_NBMAX; ++q) d[q] = cmk(0.0, 0.0);
      for (int i = jj + tid; i < hr; i += QP_NT) {
        const cplx v = i == jj ? cmk(1.0, 0.0) : P[i + jj * hr];
#pragma unroll
        for (int q = 0; q < QP_NBMAX; ++q)
          if (q < nrest) d[q] = cadd(d[q], cmulc(v, P[i + (jj + 1 + q) * hr]));
      }
#pragma unroll
      for (int q = 0; q < QP_NBMAX; ++q) {
        if (q < nrest) {
          cplx s = warp_csum(d[q]);
          if (lane == 0) sred[warp][q] = s;
        }
      }
      __syncthreads();
      if (tid < nrest) {
        cplx s = cmk(0.0, 0.0);
        for (int w = 0; w < QP_NT / 32; ++w) s = cadd(s, sred[w][tid]);
        dots[tid] = cscale(s, tau[jj]);
      }
      __syncthreads();
      for (int e = tid; e < (hr - jj) * nrest; e += QP_NT) {
        const int i = jj + e % (hr - jj), q = e / (hr - jj);
        const cplx v = i == jj ? cmk(1.0, 0.0) : P[i + jj * hr];
        P[i + (jj + 1 + q) * hr] = cfms(dots[q], v, P[i + (jj + 1 + q) * hr]);
      }
      __syncthreads();
    }
  }
  // R rows back to A (upper triangle of the panel's top jb rows)
  for (int e = tid; e < jb * jb; e += QP_NT) {
    const int i = e % jb, jj = e / jb;
    if (i <= jj) A[(j0 + i) + (size_t)(j0 + jj) * c.lda] = P[i + jj * hr];
  }
  // explicit V (unit diagonal, zeros above) and G = Vᴴ V
  cplx* V = c.V;
  for (int e = tid; e < hr * jb; e += QP_NT) {
    const int i = e % hr, jj = e / hr;
    V[i + (size_t)jj * c.h] = i < jj ? cmk(0.0, 0.0) : (i == jj ? cmk(1.0, 0.0) : P[i + jj * hr]);
  }
  {
    // 4 threads per (p, q) pair with p < q; rows strided
    const int pair = tid >> 2, part = tid & 3;
    const int npairs = jb * (jb - 1) / 2;
    for (int pb = 0; pb < npairs; pb += QP_NT / 4) {
      const int pr = pb + pair;
      cplx s = cmk(0.0, 0.0);
      int p = 0, q = 0;
      if (pr < npairs) {
        // decode pr -> (p, q), p < q
        int rem = pr;
        q = 1;
        while (rem >= q) {
          rem -= q;
          ++q;
        }
        p = rem;
        for (int i = q + part; i < hr; i += 4) {
          const cplx vp = i == p ? cmk(1.0, 0.0) : (i < p ? cmk(0.0, 0.0) : P[i + p * hr]);
          const cplx vq = i == q ? cmk(1.0, 0.0) : P[i + q * hr];
          s = cadd(s, cmulc(vp, vq));
        }
      }
      s.x += __shfl_xor_sync(0xffffffffu, s.x, 1);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, 1);
      s.x += __shfl_xor_sync(0xffffffffu, s.x, 2);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, 2);
      if (pr < npairs && part == 0) G[p][q] = s;
    }
  }
  __syncthreads();
  // T (upper triangular): T_ii = τ_i, T(0:i, i) = −τ_i T(0:i,0:i) G(0:i, i)
  if (warp == 0) {
    for (int i = 0; i < jb; ++i) {
      cplx t = cmk(0.0, 0.0);
      if (lane < i) {
        for (int q = lane; q < i; ++q) t = cfma(Tm[lane][q], G[q][i], t);
        t = cscale(t, -tau[i]);
      }
      __syncwarp();
      if (lane < i) Tm[lane][i] = t;
      if (lane == i) Tm[i][i] = cmk(tau[i], 0.0);
      if (lane > i && lane < jb) Tm[lane][i] = cmk(0.0, 0.0);
      __syncwarp();
    }
  }
  __syncthreads();
  // Z = V Tᴴ :  Z[i][cc] = Σ_{p ≥ cc} V[i][p] conj(T[cc][p])
  cplx* Z = c.Z;
  for (int e = tid; e < hr * jb; e += QP_NT) {
    const int i = e % hr, cc = e / hr;
    cplx s = cmk(0.0, 0.0);
    for (int p = cc; p < jb && p <= i; ++p) {
      const cplx v = i == p ? cmk(1.0, 0.0) : P[i + p * hr];
      const cplx tc = cmk(Tm[cc][p].x, -Tm[cc][p].y);
      s = cfma(v, tc, s);
    }
    Z[i + (size_t)cc * c.h] = s;
  }
  // zero W (jb × (b − j0 − jb)) for the next GEMM's accumulation
  cplx* W = c.W;
  const int nt = c.b - j0 - jb;
  for (int e = tid; e < NB * nt; e += QP_NT) W[e] = cmk(0.0, 0.0);
}

// ------------------------------------------------------------------ CPQR
constexpr int QR_NT = 512;

__global__ void __launch_bounds__(QR_NT) k_cpqr(const IdTask* __restrict__ tasks, cplx* ws,
                                                int* __restrict__ perm_out, int* __restrict__ k_out,
                                                double eps) {
  extern __shared__ double shm[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  const IdTask t = tasks[blockIdx.x];
  cplx* M = ws + t.M;
  const int m = t.m, b = t.b;
  double* vn1 = shm;
  double* vn2 = shm + b;
  int* perm = reinterpret_cast<int*>(shm + 2 * b);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = QR_NT / 32;
  const double tol3z = sqrt(DBL_EPSILON);

  for (int c = warp; c < b; c += nw) {
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s += cabs2(M[i + (size_t)c * m]);
    s = warp_sum(s);
    if (lane == 0) {
      vn1[c] = vn2[c] = sqrt(s);
      perm[c] = c;
    }
  }
  __syncthreads();
  const int kmax = min(m, b);
  int kk = kmax;
  double norm0 = 0.0;
  for (int j = 0; j < kmax; ++j) {
    double pv = -1.0;
    int p = INT_MAX;
    for (int c = j + tid; c < b; c += QR_NT) argmax_merge(pv, p, vn1[c], c);
    block_argmax<QR_NT>(pv, p, red_v, red_i);
    if (j == 0) norm0 = pv;
    if (!(pv > eps * norm0) || pv == 0.0) {
      kk = j;
      break;
    }
    if (p != j) {
      for (int i = tid; i < m; i += QR_NT) {
        cplx a = M[i + (size_t)j * m];
        M[i + (size_t)j * m] = M[i + (size_t)p * m];
        M[i + (size_t)p * m] = a;
      }
      if (tid == 0) {
        double x = vn1[j]; vn1[j] = vn1[p]; vn1[p] = x;
        x = vn2[j]; vn2[j] = vn2[p]; vn2[p] = x;
        int q = perm[j]; perm[j] = perm[p]; perm[p] = q;
      }
      __syncthreads();
    }
    // Householder reflector H = I − τ u uᴴ with H x = β e1, β = −(α/|α|)‖x‖
    double xs = 0.0;
    for (int i = j + 1 + tid; i < m; i += QR_NT) xs += cabs2(M[i + (size_t)j * m]);
    const double xn2 = block_sum<QR_NT>(xs, red_v);
    const cplx alpha = M[j + (size_t)j * m];
    const double aa = sqrt(cabs2(alpha));
    const double nrm = sqrt(aa * aa + xn2);
    const cplx beta = aa > 0.0 ? cmk(-alpha.x / aa * nrm, -alpha.y / aa * nrm) : cmk(-nrm, 0.0);
    const cplx u0 = csub(alpha, beta);
    const double tau = 2.0 / (cabs2(u0) + xn2);
    for (int c = j + 1 + warp; c < b; c += nw) {
      cplx* Mc = M + (size_t)c * m;
      const cplx* u = M + (size_t)j * m;
      cplx d = lane == 0 ? cmulc(u0, Mc[j]) : cmk(0.0, 0.0);
      for (int i = j + 1 + lane; i < m; i += 32) d = cadd(d, cmulc(u[i], Mc[i]));
      d = warp_csum(d);
      const cplx f = cscale(d, tau);
      if (lane == 0) Mc[j] = cfms(f, u0, Mc[j]);
      for (int i = j + 1 + lane; i < m; i += 32) Mc[i] = cfms(f, u[i], Mc[i]);
      __syncwarp();
      // LAPACK-style norm downdate with recomputation on cancellation (zlaqp2)
      int recompute = 0;
      if (lane == 0 && vn1[c] != 0.0) {
        double r = sqrt(cabs2(Mc[j])) / vn1[c];
        double temp = fmax(0.0, 1.0 - r * r);
        double q = vn1[c] / vn2[c];
        double temp2 = temp * q * q;
        if (temp2 <= tol3z) recompute = 1;
        else vn1[c] *= sqrt(temp);
      }
      recompute = __shfl_sync(0xffffffffu, recompute, 0);
      if (recompute) {
        double s = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) s += cabs2(Mc[i]);
        s = warp_sum(s);
        if (lane == 0) vn1[c] = vn2[c] = sqrt(s);
      }
    }
    __syncthreads();
    if (tid == 0) M[j + (size_t)j * m] = beta;
    __syncthreads();
  }
  for (int c = tid; c < b; c += QR_NT) perm_out[t.out_off + c] = perm[c];
  if (tid == 0) k_out[blockIdx.x] = kk;
}

// T = R11⁻¹ R12, warp per column, back substitution.
__global__ void k_trsm_T(const IdTask* __restrict__ tasks, const int* __restrict__ kv,
                         const cplx* __restrict__ ws, cplx* __restrict__ tarena) {
  const IdTask t = tasks[blockIdx.x];
  const int kk = kv[blockIdx.x];
  const int r = t.b - kk, m = t.m;
  const cplx* M = ws + t.M;
  cplx* T = tarena + t.T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < r; c += nw) {
    cplx* x = T + (size_t)c * kk;
    for (int i = lane; i < kk; i += 32) x[i] = M[i + (size_t)(kk + c) * m];
    __syncwarp();
    for (int l = kk - 1; l >= 0; --l) {
      const cplx xl = cdiv(x[l], M[l + (size_t)l * m]);
      __syncwarp();
      if (lane == 0) x[l] = xl;
      for (int i = lane; i < l; i += 32) x[i] = cfms(M[i + (size_t)l * m], xl, x[i]);
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ Gauss-Jordan inverse
constexpr int GJ_NT = 512;

__global__ void __launch_bounds__(GJ_NT) k_gj(const long long* __restrict__ offs,
                                              const int* __restrict__ dims, cplx* arena,
                                              int* status) {
  extern __shared__ double shm[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  const int n = dims[blockIdx.x];
  cplx* A = arena + offs[blockIdx.x];
  cplx* colj = reinterpret_cast<cplx*>(shm);
  cplx* rowj = colj + n;
  int* piv = reinterpret_cast<int*>(rowj + n);
  const int tid = threadIdx.x;
  for (int j = 0; j < n; ++j) {
    double pv = -1.0;
    int p = INT_MAX;
    for (int i = j + tid; i < n; i += GJ_NT) argmax_merge(pv, p, cabs2(A[i + (size_t)j * n]), i);
    block_argmax<GJ_NT>(pv, p, red_v, red_i);
    if (!(pv > 0.0)) {
      if (tid == 0) atomicExch(status, 1);
      return;
    }
    if (tid == 0) piv[j] = p;
    if (p != j)
      for (int c = tid; c < n; c += GJ_NT) {
        cplx a = A[j + (size_t)c * n];
        A[j + (size_t)c * n] = A[p + (size_t)c * n];
        A[p + (size_t)c * n] = a;
      }
    __syncthreads();
    const cplx d = A[j + (size_t)j * n];
    const cplx dinv = cdiv(cmk(1.0, 0.0), d);
    for (int i = tid; i < n; i += GJ_NT) colj[i] = A[i + (size_t)j * n];
    for (int c = tid; c < n; c += GJ_NT) rowj[c] = c == j ? dinv : cmul(A[j + (size_t)c * n], dinv);
    __syncthreads();
    for (int e = tid; e < n * n; e += GJ_NT) {
      const int i = e % n, c = e / n;
      cplx v;
      if (i == j) v = rowj[c];
      else if (c == j) v = cmk(-(colj[i].x * dinv.x - colj[i].y * dinv.y), -(colj[i].x * dinv.y + colj[i].y * dinv.x));
      else v = cfms(colj[i], rowj[c], A[i + (size_t)c * n]);
      A[i + (size_t)c * n] = v;
    }
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {
    const int p = piv[j];
    if (p != j)
      for (int i = tid; i < n; i += GJ_NT) {
        cplx a = A[i + (size_t)j * n];
        A[i + (size_t)j * n] = A[i + (size_t)p * n];
        A[i + (size_t)p * n] = a;
      }
    __syncthreads();
  }
}

// Cooperative Gauss-Jordan inverse (root block D_t⁻¹): columns are
// owned round-robin by the CTAs; one grid barrier per elimination step.  Output to B
// (column permutation undone out-of-place).
constexpr int GJC_NT = 512;
__global__ void __launch_bounds__(GJC_NT) k_gj_coop(cplx* A, cplx* B, int n, cplx* scratch,
                                                    int* piv, int* status) {
  extern __shared__ double shm[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  cg::grid_group grid = cg::this_grid();
  cplx* col = reinterpret_cast<cplx*>(shm);
  const int tid = threadIdx.x, G = gridDim.x, gb = blockIdx.x;
  if (gb == 0)
    for (int i = tid; i < n; i += GJC_NT) scratch[i] = A[i];
  grid.sync();
  for (int j = 0; j < n; ++j) {
    const cplx* cj = scratch + (size_t)(j & 1) * n;
    for (int i = tid; i < n; i += GJC_NT) col[i] = cj[i];
    __syncthreads();
    double pv = -1.0;
    int p = INT_MAX;
    for (int i = j + tid; i < n; i += GJC_NT) argmax_merge(pv, p, cabs2(col[i]), i);
    block_argmax<GJC_NT>(pv, p, red_v, red_i);
    if (!(pv > 0.0)) {
      if (gb == 0 && tid == 0) atomicExch(status, 1);
      return;  // uniform across the grid (same column data everywhere)
    }
    if (gb == 0 && tid == 0) piv[j] = p;
    const cplx d = col[p];
    const cplx dinv = cdiv(cmk(1.0, 0.0), d);
    __syncthreads();
    if (tid == 0 && p != j) {  // swapped column j
      cplx a = col[j];
      col[j] = col[p];
      col[p] = a;
    }
    __syncthreads();
    for (int c = gb; c < n; c += G) {
      cplx* Ac = A + (size_t)c * n;
      cplx rj;
      if (tid == 0) {
        if (p != j) {
          cplx a = Ac[j];
          Ac[j] = Ac[p];
          Ac[p] = a;
        }
      }
      __syncthreads();
      rj = Ac[j];
      __syncthreads();
      if (c == j) {
        for (int i = tid; i < n; i += GJC_NT)
          Ac[i] = i == j ? dinv : cmk(-(col[i].x * dinv.x - col[i].y * dinv.y), -(col[i].x * dinv.y + col[i].y * dinv.x));
      } else {
        const cplx rs = cmul(rj, dinv);
        for (int i = tid; i < n; i += GJC_NT) Ac[i] = i == j ? rs : cfms(col[i], rs, Ac[i]);
      }
      if (c == j + 1) {
        __syncthreads();
        for (int i = tid; i < n; i += GJC_NT) scratch[(size_t)((j + 1) & 1) * n + i] = Ac[i];
      }
      __syncthreads();
    }
    grid.sync();
  }
  // undo the column interchanges: final column c = column L[c] (L = swaps applied in reverse)
  int* L = reinterpret_cast<int*>(shm);
  for (int c = tid; c < n; c += GJC_NT) L[c] = c;
  __syncthreads();
  if (tid == 0)
    for (int j = n - 1; j >= 0; --j) {
      int p = piv[j];
      int a = L[j];
      L[j] = L[p];
      L[p] = a;
    }
  __syncthreads();
  for (int c = gb; c < n; c += G) {
    const cplx* src = A + (size_t)L[c] * n;
    for (int i = tid; i < n; i += GJC_NT) B[i + (size_t)c * n] = src[i];
  }
}

// ------------------------------------------------------------------ solve sweeps
constexpr int SV_NT = 256;
constexpr int SV_Q = 4;  // RHS processed per pass

__global__ void __launch_bounds__(SV_NT) k_solve_up(const BoxRec* __restrict__ recs,
                                                    const cplx* __restrict__ fac,
                                                    const int* __restrict__ idx, cplx* y, int ldy,
                                                    int nrhs) {
  extern __shared__ double shm[];
  const BoxRec R = recs[blockIdx.x];
  const int k = R.k, r = R.r, nN = R.nN, kn = k + nN;
  cplx* yS = reinterpret_cast<cplx*>(shm);  // k × Q
  cplx* yR = yS + k * SV_Q;                // r × Q
  cplx* tmp = yR + r * SV_Q;               // r × Q
  const int* S = idx + R.idxS;
  const int* Ri = idx + R.idxR;
  const int* N = idx + R.idxN;
  const cplx* T = fac + R.T;
  const cplx* Xi = fac + R.Xi;
  const cplx* Lp = fac + R.Lp;
  for (int q0 = 0; q0 < nrhs; q0 += SV_Q) {
    const int nq = min(SV_Q, nrhs - q0);
    for (int e = threadIdx.x; e < k * nq; e += SV_NT) {
      int i = e % k, q = e / k;
      yS[i + q * k] = y[S[i] + (size_t)(q0 + q) * ldy];
    }
    for (int e = threadIdx.x; e < r * nq; e += SV_NT) {
      int i = e % r, q = e / r;
      yR[i + q * r] = y[Ri[i] + (size_t)(q0 + q) * ldy];
    }
    __syncthreads();
    // E: y_R −= Tᵀ y_S
    for (int e = threadIdx.x; e < r * nq; e += SV_NT) {
      int i = e % r, q = e / r;
      cplx v = yR[i + q * r];
      for (int l = 0; l < k; ++l) v = cfms(T[l + (size_t)i * k], yS[l + q * k], v);
      tmp[i + q * r] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < r * nq; e += SV_NT) yR[e] = tmp[e];
    __syncthreads();
    // L: y_{S∪N} −= Lp y_R  (N rows shared with other boxes of the phase → atomics)
    for (int f = threadIdx.x; f < kn; f += SV_NT) {
      cplx acc[SV_Q];
#pragma unroll
      for (int q = 0; q < SV_Q; ++q) acc[q] = cmk(0.0, 0.0);
      for (int i = 0; i < r; ++i) {
        const cplx l = Lp[f + (size_t)i * kn];
#pragma unroll
        for (int q = 0; q < SV_Q; ++q)
          if (q < nq) acc[q] = cfma(l, yR[i + q * r], acc[q]);
      }
      for (int q = 0; q < nq; ++q) {
        if (f < k) {
          yS[f + q * k] = csub(yS[f + q * k], acc[q]);
        } else {
          cplx* d = y + N[f - k] + (size_t)(q0 + q) * ldy;
          atomicAdd(&d->x, -acc[q].x);
          atomicAdd(&d->y, -acc[q].y);
        }
      }
    }
    // D⁻¹ on R: y_R ← X_RR⁻¹ y_R
    for (int e = threadIdx.x; e < r * nq; e += SV_NT) {
      int i = e % r, q = e / r;
      cplx v = cmk(0.0, 0.0);
      for (int l = 0; l < r; ++l) v = cfma(Xi[i + (size_t)l * r], yR[l + q * r], v);
      tmp[i + q * r] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * nq; e += SV_NT) {
      int i = e % k, q = e / k;
      y[S[i] + (size_t)(q0 + q) * ldy] = yS[i + q * k];
    }
    for (int e = threadIdx.x; e < r * nq; e += SV_NT) {
      int i = e % r, q = e / r;
      y[Ri[i] + (size_t)(q0 + q) * ldy] = tmp[i + q * r];
    }
    __syncthreads();
  }
}

constexpr int SV_FCH = 1024;  // S∪N entries staged per chunk in the downward sweep
__global__ void __launch_bounds__(SV_NT) k_solve_down(const BoxRec* __restrict__ recs,
                                                      const cplx* __restrict__ fac,
                                                      const int* __restrict__ idx, cplx* y,
                                                      int ldy, int nrhs) {
  extern __shared__ double shm[];
  const BoxRec R = recs[blockIdx.x];
  const int k = R.k, r = R.r, nN = R.nN, kn = k + nN;
  cplx* ySN = reinterpret_cast<cplx*>(shm);  // SV_FCH × Q
  cplx* yR = ySN + SV_FCH * SV_Q;            // r × Q
  const int* S = idx + R.idxS;
  const int* Ri = idx + R.idxR;
  const int* N = idx + R.idxN;
  const cplx* T = fac + R.T;
  const cplx* Up = fac + R.Up;
  for (int q0 = 0; q0 < nrhs; q0 += SV_Q) {
    const int nq = min(SV_Q, nrhs - q0);
    for (int e = threadIdx.x; e < r * nq; e += SV_NT) {
      int i = e % r, q = e / r;
      yR[i + q * r] = y[Ri[i] + (size_t)(q0 + q) * ldy];
    }
    // U: y_R −= Up y_{S∪N}, S∪N staged in chunks
    for (int f0 = 0; f0 < kn; f0 += SV_FCH) {
      const int fn = min(SV_FCH, kn - f0);
      __syncthreads();
      for (int e = threadIdx.x; e < fn * nq; e += SV_NT) {
        int f = e % fn, q = e / fn;
        int gi = (f0 + f) < k ? S[f0 + f] : N[f0 + f - k];
        ySN[f + q * SV_FCH] = y[gi + (size_t)(q0 + q) * ldy];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < r * nq; e += SV_NT) {
        int i = e % r, q = e / r;
        cplx v = yR[i + q * r];
        for (int f = 0; f < fn; ++f) v = cfms(Up[i + (size_t)(f0 + f) * r], ySN[f + q * SV_FCH], v);
        yR[i + q * r] = v;
      }
    }
    __syncthreads();
    // F: y_S −= T y_R
    for (int e = threadIdx.x; e < k * nq; e += SV_NT) {
      int l = e % k, q = e / k;
      cplx v = y[S[l] + (size_t)(q0 + q) * ldy];
      for (int i = 0; i < r; ++i) v = cfms(T[l + (size_t)i * k], yR[i + q * r], v);
      y[S[l] + (size_t)(q0 + q) * ldy] = v;
    }
    for (int e = threadIdx.x; e < r * nq; e += SV_NT) {
      int i = e % r, q = e / r;
      y[Ri[i] + (size_t)(q0 + q) * ldy] = yR[i + q * r];
    }
    __syncthreads();
  }
}

// root: tmp = y[rows]; y[rows] = Xinv · tmp   (one thread per row, column-major Xinv)
__global__ void k_root_gather(const int* rows, const cplx* y, int ldy, cplx* tmp, int n0, int nrhs) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n0 * nrhs; e += gridDim.x * blockDim.x) {
    int i = e % n0, q = e / n0;
    tmp[e] = y[rows[i] + (size_t)q * ldy];
  }
}
__global__ void k_root_apply(const cplx* __restrict__ Xi, int n0, const int* __restrict__ rows,
                             cplx* y, int ldy, int nrhs, const cplx* __restrict__ tmp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (int q0 = 0; q0 < nrhs; q0 += SV_Q) {
    const int nq = min(SV_Q, nrhs - q0);
    if (i < n0) {
      cplx acc[SV_Q];
#pragma unroll
      for (int q = 0; q < SV_Q; ++q) acc[q] = cmk(0.0, 0.0);
      for (int l = 0; l < n0; ++l) {
        const cplx a = Xi[i + (size_t)l * n0];
#pragma unroll
        for (int q = 0; q < SV_Q; ++q)
          if (q < nq) acc[q] = cfma(a, tmp[l + (size_t)(q0 + q) * n0], acc[q]);
      }
      for (int q = 0; q < nq; ++q) y[rows[i] + (size_t)(q0 + q) * ldy] = acc[q];
    }
  }
}

// ------------------------------------------------------------------ permutes
// mode 1: dst[i] = src[perm[i]] * sw[i]    (caller → tree order, W^{½})
// mode 0: plain permutation
__global__ void k_perm_in(const cplx* src, int ld_src, cplx* dst, int n, int nrhs,
                          const long long* perm, const double* sw, int mode) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * nrhs;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e % n), q = (int)(e / n);
    cplx v = src[perm[i] + (size_t)q * ld_src];
    if (mode) v = cscale(v, sw[i]);
    dst[e] = v;
  }
}
__global__ void k_perm_out(const cplx* src, cplx* dst, int ld_dst, int n, int nrhs,
                           const long long* perm, const double* sw, int mode) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * nrhs;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e % n), q = (int)(e / n);
    cplx v = src[e];
    if (mode) v = cscale(v, 1.0 / sw[i]);
    dst[perm[i] + (size_t)q * ld_dst] = v;
  }
}

// ------------------------------------------------------------------ brute-force matvec
constexpr int MV_NT = 128;
constexpr int MV_Q = 4;
__global__ void __launch_bounds__(MV_NT) k_matvec(Geo g, double k, int n, const cplx* __restrict__ x,
                                                  cplx* __restrict__ y, int nrhs, int q0) {
  __shared__ double sx[MV_NT], sy[MV_NT], sz[MV_NT], snx[MV_NT], sny[MV_NT], snz[MV_NT];
  __shared__ cplx swx[MV_Q][MV_NT];
  const int i = blockIdx.x * MV_NT + threadIdx.x;
  const int nq = min(MV_Q, nrhs - q0);
  double xi = 0, yi = 0, zi = 0;
  if (i < n) {
    xi = g.x[i];
    yi = g.y[i];
    zi = g.z[i];
  }
  cplx acc[MV_Q];
#pragma unroll
  for (int q = 0; q < MV_Q; ++q) acc[q] = cmk(0.0, 0.0);
  for (int j0 = 0; j0 < n; j0 += MV_NT) {
    const int j = j0 + threadIdx.x;
    if (j < n) {
      sx[threadIdx.x] = g.x[j];
      sy[threadIdx.x] = g.y[j];
      sz[threadIdx.x] = g.z[j];
      snx[threadIdx.x] = g.nx[j];
      sny[threadIdx.x] = g.ny[j];
      snz[threadIdx.x] = g.nz[j];
      const double w = g.sw[j] * g.sw[j];
#pragma unroll
      for (int q = 0; q < MV_Q; ++q)
        swx[q][threadIdx.x] = q < nq ? cscale(x[j + (size_t)(q0 + q) * n], w) : cmk(0.0, 0.0);
    }
    __syncthreads();
    const int jn = min(MV_NT, n - j0);
    if (i < n)
      for (int jj = 0; jj < jn; ++jj) {
        if (j0 + jj == i) continue;
        const cplx K = kernel_K(k, xi - sx[jj], yi - sy[jj], zi - sz[jj], snx[jj], sny[jj], snz[jj]);
#pragma unroll
        for (int q = 0; q < MV_Q; ++q) acc[q] = cfma(K, swx[q][jj], acc[q]);
      }
    __syncthreads();
  }
  if (i < n)
    for (int q = 0; q < nq; ++q) {
      const cplx xv = x[i + (size_t)(q0 + q) * n];
      y[i + (size_t)(q0 + q) * n] = cadd(acc[q], cscale(xv, 0.5));
    }
}

// ------------------------------------------------------------------ FP64 probes
__global__ void k_probe_dfma(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_probe_dmma(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

// ------------------------------------------------------------------ launchers
void launch_build(const BuildTask* d_tasks, int ntasks, const int* gidx, const int* slot,
                  const int* pos, const long long* tab, const int* bld, const cplx* src_arena,
                  cplx* dst_arena, const Geo& g, double k, cudaStream_t st) {
  if (ntasks <= 0) return;
  k_build<<<ntasks, 256, 0, st>>>(d_tasks, gidx, slot, pos, tab, bld, src_arena, dst_arena, g, k);
  FMMLU_LAUNCH();
}

void launch_copy(const CopyTask* d_tasks, int ntasks, const int* maps, const cplx* src_arena,
                 cplx* dst_arena, cudaStream_t st) {
  if (ntasks <= 0) return;
  k_copy<<<ntasks, 256, 0, st>>>(d_tasks, maps, src_arena, dst_arena);
  FMMLU_LAUNCH();
}

void launch_proxy(const ProxyTask* d_tasks, int ntasks, const int* gidx, cplx* ws, const Geo& g,
                  double k, cudaStream_t st) {
  if (ntasks <= 0) return;
  dim3 grid(ntasks, 8);
  k_proxy<<<grid, 256, 0, st>>>(d_tasks, gidx, ws, g, k);
  FMMLU_LAUNCH();
}

void launch_qr_panel(const QrChunk* d_chunks, int nchunks, int j0, int nb, cudaStream_t st) {
  if (nchunks <= 0) return;
  static bool init = false;
  if (!init) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_qr_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    init = true;
  }
  k_qr_panel<<<nchunks, QP_NT, 200 * 1024, st>>>(d_chunks, j0, nb);
  FMMLU_LAUNCH();
}

void launch_cpqr(const IdTask* d_tasks, int ntasks, cplx* ws, int* perm_out, int* k_out,
                 double eps, cudaStream_t st, int bmax) {
  if (ntasks <= 0) return;
  size_t smem = (size_t)bmax * (2 * sizeof(double) + sizeof(int)) + 16;
  static size_t cur = 0;
  if (smem > 48 * 1024 && smem > cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_cpqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  k_cpqr<<<ntasks, QR_NT, smem, st>>>(d_tasks, ws, perm_out, k_out, eps);
  FMMLU_LAUNCH();
}


void launch_trsm_T(const IdTask* d_tasks, const int* d_k, int ntasks, const cplx* ws,
                   cplx* tarena, cudaStream_t st) {
  if (ntasks <= 0) return;
  k_trsm_T<<<ntasks, 512, 0, st>>>(d_tasks, d_k, ws, tarena);
  FMMLU_LAUNCH();
}

void launch_gj_inverse(const long long* d_off, const int* d_dim, int nmat, cplx* arena,
                       int* d_status, cudaStream_t st, int nmax) {
  if (nmat <= 0) return;
  size_t smem = (size_t)nmax * (2 * sizeof(cplx) + sizeof(int)) + 16;
  static size_t cur = 0;
  if (smem > 48 * 1024 && smem > cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_gj, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  k_gj<<<nmat, GJ_NT, smem, st>>>(d_off, d_dim, arena, d_status);
  FMMLU_LAUNCH();
}


void launch_gj_inverse_coop(cplx* A, int n, cplx* scratch, int* d_status, cudaStream_t st) {
  // scratch: 2n complex (column buffers) + n ints (pivots) + n*n complex (output)
  int dev;
  FMMLU_CUDA(cudaGetDevice(&dev));
  int nsm;
  FMMLU_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  size_t smem = (size_t)n * sizeof(cplx) + 16;
  FMMLU_CUDA(cudaFuncSetAttribute(k_gj_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  FMMLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gj_coop, GJC_NT, smem));
  if (per_sm < 1) throw Error(-4, "root block too large for the cooperative GJ kernel");
  int G = nsm;
  cplx* colbuf = scratch;
  int* piv = reinterpret_cast<int*>(scratch + 2 * (size_t)n);
  cplx* B = scratch + 2 * (size_t)n + (n + 1) / 2 + 1;
  void* args[] = {&A, &B, &n, &colbuf, &piv, &d_status};
  FMMLU_CUDA(cudaLaunchCooperativeKernel((void*)k_gj_coop, G, GJC_NT, args, smem, st));
  FMMLU_LAUNCH();
  FMMLU_CUDA(cudaMemcpyAsync(A, B, (size_t)n * n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
}

void launch_solve_up(const BoxRec* d_recs, int nrec, const cplx* fac, const int* idx, cplx* y,
                     int ldy, int nrhs, cudaStream_t st, int kmax, int rmax) {
  if (nrec <= 0) return;
  size_t smem = (size_t)(kmax + 2 * rmax) * SV_Q * sizeof(cplx) + 16;
  static size_t cur = 0;
  if (smem > 48 * 1024 && smem > cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_solve_up, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  k_solve_up<<<nrec, SV_NT, smem, st>>>(d_recs, fac, idx, y, ldy, nrhs);
  FMMLU_LAUNCH();
}

void launch_solve_down(const BoxRec* d_recs, int nrec, const cplx* fac, const int* idx, cplx* y,
                       int ldy, int nrhs, cudaStream_t st, int rmax) {
  if (nrec <= 0) return;
  size_t smem = (size_t)(SV_FCH + rmax) * SV_Q * sizeof(cplx) + 16;
  static size_t cur = 0;
  if (smem > 48 * 1024 && smem > cur) {
    FMMLU_CUDA(cudaFuncSetAttribute(k_solve_down, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  k_solve_down<<<nrec, SV_NT, smem, st>>>(d_recs, fac, idx, y, ldy, nrhs);
  FMMLU_LAUNCH();
}


void launch_root_apply(const cplx* Xinv, int n0, const int* d_rows, cplx* y, int ldy, int nrhs,
                       cplx* tmp, cudaStream_t st) {
  if (n0 <= 0) return;
  k_root_gather<<<256, 256, 0, st>>>(d_rows, y, ldy, tmp, n0, nrhs);
  FMMLU_LAUNCH();
  k_root_apply<<<(n0 + 127) / 128, 128, 0, st>>>(Xinv, n0, d_rows, y, ldy, nrhs, tmp);
  FMMLU_LAUNCH();
}

void launch_permute_in(const cplx* src, int ld_src, cplx* dst, int n, int nrhs,
                       const long long* perm, const double* sw, int mode, cudaStream_t st) {
  k_perm_in<<<592, 256, 0, st>>>(src, ld_src, dst, n, nrhs, perm, sw, mode);
  FMMLU_LAUNCH();
}
void launch_permute_out(const cplx* src, cplx* dst, int ld_dst, int n, int nrhs,
                        const long long* perm, const double* sw, int mode, cudaStream_t st) {
  k_perm_out<<<592, 256, 0, st>>>(src, dst, ld_dst, n, nrhs, perm, sw, mode);
  FMMLU_LAUNCH();
}

void launch_matvec(const Geo& g, double k, int n, const cplx* x, cplx* y, int nrhs,
                   cudaStream_t st) {
  for (int q0 = 0; q0 < nrhs; q0 += MV_Q) {
    k_matvec<<<(n + MV_NT - 1) / MV_NT, MV_NT, 0, st>>>(g, k, n, x, y, nrhs, q0);
    FMMLU_LAUNCH();
  }
}

double probe_fp64(int kind) {
  int dev, nsm;
  FMMLU_CUDA(cudaGetDevice(&dev));
  FMMLU_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double* out;
  FMMLU_CUDA(cudaMalloc(&out, 8));
  const int iters = 4096, blocks = nsm * 8, threads = 256;
  cudaEvent_t a, b;
  FMMLU_CUDA(cudaEventCreate(&a));
  FMMLU_CUDA(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    FMMLU_CUDA(cudaEventRecord(a));
    if (kind == 0) k_probe_dfma<<<blocks, threads>>>(out, iters);
    else k_probe_dmma<<<blocks, threads>>>(out, iters);
    FMMLU_CUDA(cudaEventRecord(b));
    FMMLU_CUDA(cudaEventSynchronize(b));
    float ms;
    FMMLU_CUDA(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  double flops = kind == 0 ? 2.0 * 8 * iters * (double)blocks * threads
                           : 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace fmmlu
