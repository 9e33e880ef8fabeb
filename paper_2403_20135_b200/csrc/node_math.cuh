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
// both components (re, im) of coefficient idx: 16-byte accesses
__device__ __forceinline__ void load_tri2(const double* __restrict__ s, int C, int idx, Tri& re,
                                          Tri& im) {
  const double2* q = reinterpret_cast<const double2*>(s);
  const double2 a = q[idx], b = q[C + idx], c = q[2 * C + idx];
  re = Tri{a.x, b.x, c.x};
  im = Tri{a.y, b.y, c.y};
}
__device__ __forceinline__ void store_tri2(double* __restrict__ s, int C, int idx, const Tri& re,
                                           const Tri& im) {
  double2* q = reinterpret_cast<double2*>(s);
  q[idx] = make_double2(re.phi, im.phi);
  q[C + idx] = make_double2(re.zeta, im.zeta);
  q[2 * C + idx] = make_double2(re.delta, im.delta);
}
// the whole synthesis-operand record of one coefficient (both components):
// three 32-byte chunks, values as write_xsyn_half (internal.cuh) computes them
__device__ __forceinline__ void write_xsyn_full(double* __restrict__ rec, size_t pstride,
                                                const Tri& re, const Tri& im, double2 sc) {
  const double sm = sc.x, sa = sc.y;
  double2* p0 = reinterpret_cast<double2*>(rec);
  double2* p1 = reinterpret_cast<double2*>(rec + pstride);
  double2* p2 = reinterpret_cast<double2*>(rec + 2 * pstride);
#if SDCSW_MUTATE_UCHI  // test-only mutation: wrong sign of the i m chi term of U (KAT proof)
  p0[0] = make_double2(-sm * im.delta, sm * re.delta);
#else
  p0[0] = make_double2(sm * im.delta, -sm * re.delta);  // U_P re, im
#endif
  p0[1] = make_double2(sm * im.zeta, -sm * re.zeta);    // V_P re, im
  p1[0] = make_double2(re.zeta, im.zeta);
  p1[1] = make_double2(re.phi, im.phi);
  p2[0] = make_double2(sa * re.zeta, sa * im.zeta);     // U_H
  p2[1] = make_double2(-sa * re.delta, -sa * im.delta); // V_H
}
__device__ __forceinline__ bool finite_tri(const Tri& t) {
  return isfinite(t.phi) && isfinite(t.zeta) && isfinite(t.delta);
}


}  // namespace sdcsw
