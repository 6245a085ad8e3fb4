// Shared device helpers for libfmmlu (complex fp64 arithmetic, the
// combined-field kernel entry, launch checks).  Product code only — nothing
// here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

typedef double2 cplx;  // (re, im), layout-compatible with cuDoubleComplex / complex128

#include "error.h"

namespace fmmlu {

#define FMMLU_CUDA(call)                                                              \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw ::fmmlu::Error(-7, std::string(#call) + ": " + cudaGetErrorString(e_) +   \
                                   " @" + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define FMMLU_LAUNCH() FMMLU_CUDA(cudaGetLastError())

__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ __forceinline__ cplx cmulc(cplx a, cplx b) {
  return cmk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return cmk(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return cmk(a.x, -a.y); }
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  // Smith-free straightforward division (b well away from 0/inf in our use)
  double d = 1.0 / (b.x * b.x + b.y * b.y);
  return cmk((a.x * b.x + a.y * b.y) * d, (a.y * b.x - a.x * b.y) * d);
}
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {  // c + a*b
  return cmk(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ cplx cfms(cplx a, cplx b, cplx c) {  // c - a*b
  return cmk(fma(-a.x, b.x, fma(a.y, b.y, c.x)), fma(-a.x, b.y, fma(-a.y, b.x, c.y)));
}

constexpr double kInv4Pi = 0.079577471545947667884441881686257181;  // 1/(4π)

// Combined-field kernel K(x, y) = n(y)·∇_y G(x,y) − ik G(x,y) (PAPER.md Eq. comb_ref,
// L414-421; reading C2): e^{ikr}(1−ikr)((x−y)·n(y))/(4πr³) − ik e^{ikr}/(4πr).
__device__ __forceinline__ cplx kernel_K(double k, double dx, double dy, double dz, double nx,
                                         double ny, double nz) {
  double r2 = dx * dx + dy * dy + dz * dz;
  double rinv = rsqrt(r2);
  // refine rsqrt to full fp64 accuracy (one Newton step)
  rinv = rinv * (1.5 - 0.5 * r2 * rinv * rinv);
  double r = r2 * rinv;
  double s, c;
  sincos(k * r, &s, &c);
  double g = kInv4Pi * rinv;            // 1/(4πr)
  double dn = dx * nx + dy * ny + dz * nz;  // (x−y)·n(y)
  double f = dn * rinv * rinv;          // (x−y)·n/r²
  // D = e^{ikr}(1 − ikr) f g ; S = e^{ikr} g ; K = D − ik S
  // e^{ikr}(1−ikr) = (c + i s)(1 − i kr) = (c + s kr) + i (s − c kr)
  double kr = k * r;
  double dre = (c + s * kr) * f * g, dim = (s - c * kr) * f * g;
  // −ik e^{ikr} g = −ik(c + i s) g = (k s g) + i(−k c g)
  return cmk(dre + k * s * g, dim - k * c * g);
}

// Single layer G(x, y) = e^{ikr}/(4πr) (PAPER.md Eq. greenfunhelm).
__device__ __forceinline__ cplx kernel_G(double k, double dx, double dy, double dz) {
  double r2 = dx * dx + dy * dy + dz * dz;
  double rinv = rsqrt(r2);
  rinv = rinv * (1.5 - 0.5 * r2 * rinv * rinv);
  double r = r2 * rinv;
  double s, c;
  sincos(k * r, &s, &c);
  double g = kInv4Pi * rinv;
  return cmk(c * g, s * g);
}

// Device-resident geometry in tree order (SoA).
struct Geo {
  const double* x;
  const double* y;
  const double* z;
  const double* nx;
  const double* ny;
  const double* nz;
  const double* sw;  // √w
};

// Scaled matrix entry Ã_ij = √w_i K(x_i,x_j) √w_j (i≠j), ½ (i=j) (PAPER.md Eq. disc3; C1/C19).
__device__ __forceinline__ cplx entry_scaled(const Geo& g, double k, int i, int j) {
  if (i == j) return cmk(0.5, 0.0);
  cplx K = kernel_K(k, g.x[i] - g.x[j], g.y[i] - g.y[j], g.z[i] - g.z[j], g.nx[j], g.ny[j],
                    g.nz[j]);
  return cscale(K, g.sw[i] * g.sw[j]);
}

}  // namespace fmmlu
