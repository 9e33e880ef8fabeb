// Node arithmetic shared by the node kernels (nodes.cu) and the sweep-fused
// analysis epilogue (legendre.cu): explicitly rounded IEEE operations in the
// order numpy evaluates the reference expressions (bit-identical results).
#pragma once
#include "internal.cuh"

namespace sdcsw {

struct NodeArgs {
  double v[16 * 20];
};

// A thread owns one real component (re or im) of one coefficient index across
// the three fields; the solve and f_I are component-wise (all coefficients are
// real), so this is bit-identical to the complex formulation and doubles the
// parallelism.  Element e in [0, 2C) of field f lives at double offset f*2C + e.
struct Tri {
  double phi, zeta, delta;
};

__device__ __forceinline__ Tri load_tri(const double* __restrict__ s, int C2, int e) {
  Tri t;
  t.phi = s[e];
  t.zeta = s[C2 + e];
  t.delta = s[2 * C2 + e];
  return t;
}
__device__ __forceinline__ void store_tri(double* __restrict__ s, int C2, int e, const Tri& t) {
  s[e] = t.phi;
  s[C2 + e] = t.zeta;
  s[2 * C2 + e] = t.delta;
}
__device__ __forceinline__ double axpy1(double acc, double w, double x) {
  return __dadd_rn(acc, __dmul_rn(w, x));
}
__device__ __forceinline__ double axmy1(double acc, double w, double x) {
  return __dsub_rn(acc, __dmul_rn(w, x));
}
__device__ __forceinline__ Tri axpy_tri(Tri a, double w, const Tri& x) {
  a.phi = axpy1(a.phi, w, x.phi);
  a.zeta = axpy1(a.zeta, w, x.zeta);
  a.delta = axpy1(a.delta, w, x.delta);
  return a;
}
__device__ __forceinline__ Tri axmy_tri(Tri a, double w, const Tri& x) {
  a.phi = axmy1(a.phi, w, x.phi);
  a.zeta = axmy1(a.zeta, w, x.zeta);
  a.delta = axmy1(a.delta, w, x.delta);
  return a;
}
__device__ __forceinline__ Tri add_tri(const Tri& a, const Tri& b) {
  return Tri{__dadd_rn(a.phi, b.phi), __dadd_rn(a.zeta, b.zeta), __dadd_rn(a.delta, b.delta)};
}
__device__ __forceinline__ Tri sub_tri(const Tri& a, const Tri& b) {
  return Tri{__dsub_rn(a.phi, b.phi), __dsub_rn(a.zeta, b.zeta), __dsub_rn(a.delta, b.delta)};
}
// f_I(u) = (-phibar delta, 0, lam phi)
__device__ __forceinline__ Tri f_impl_tri(const Tri& u, double phibar, double lam) {
  return Tri{__dmul_rn(-phibar, u.delta), 0.0, __dmul_rn(lam, u.phi)};
}
// u - alpha f_I(u) = beta:  phi = (b_phi - a_phi b_delta) * inv,
// inv = 1 / (1 + a2_phi lam), zeta = b_zeta, delta = b_delta + (alpha lam) phi
__device__ __forceinline__ Tri solve_tri(const Tri& b, double alpha, double a_phi, double a2_phi,
                                         double lam) {
  const double inv = __ddiv_rn(1.0, __dadd_rn(1.0, __dmul_rn(a2_phi, lam)));
  Tri u;
  u.phi = __dmul_rn(axmy1(b.phi, a_phi, b.delta), inv);
  u.zeta = b.zeta;
  u.delta = axpy1(b.delta, __dmul_rn(alpha, lam), u.phi);
  return u;
}
__device__ __forceinline__ bool finite_tri(const Tri& t) {
  return isfinite(t.phi) && isfinite(t.zeta) && isfinite(t.delta);
}


}  // namespace sdcsw
