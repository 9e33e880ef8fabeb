// Small-DFT building blocks shared by the ring FFT (ring_fft.cu) and the
// planar 2-D FFTs (planar.cu): complex helpers and in-register radix-2/3/4/8/16
// butterflies (INV: exp(+i...), else exp(-i...)).
#pragma once
#include "internal.cuh"

namespace sdcsw {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
  const double2 s13 = cadd(a1, a3), d13 = rot<INV>(csub(a1, a3));
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, d13);
  a3 = csub(d02, d13);
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2 (&u)[R]) {
  if constexpr (R == 2) {
    const double2 a = u[0], b = u[1];
    u[0] = cadd(a, b);
    u[1] = csub(a, b);
  } else if constexpr (R == 3) {
    const double s3 = 0.86602540378443864676;  // sqrt(3)/2
    const double2 t1 = cadd(u[1], u[2]);
    const double2 t2 = make_double2(u[0].x - 0.5 * t1.x, u[0].y - 0.5 * t1.y);
    const double2 d = csub(u[1], u[2]);
    const double2 isd = rot<INV>(make_double2(s3 * d.x, s3 * d.y));  // -i s d (fwd)
    u[0] = cadd(u[0], t1);
    u[1] = cadd(t2, isd);
    u[2] = csub(t2, isd);
  } else if constexpr (R == 4) {
    dft4<INV>(u[0], u[1], u[2], u[3]);
  } else if constexpr (R == 16) {
    // 16 = 4 x 4: X_b[c] = DFT4_a(u[4a + b]); X_b[c] *= w16^(b c); y[c + 4d] = DFT4_b(X_b[c])
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
    constexpr double H = 0.70710678118654752440;
    // cos / sin of 2 pi e / 16 for e = 0..9
    constexpr double cs[10][2] = {{1, 0},   {C1, S1}, {H, H},     {S1, C1},   {0, 1},
                                  {-S1, C1}, {-H, H}, {-C1, S1}, {-1, 0},   {-C1, -S1}};
#pragma unroll
    for (int b = 0; b < 4; ++b) dft4<INV>(u[b], u[4 + b], u[8 + b], u[12 + b]);
#pragma unroll
    for (int b = 1; b < 4; ++b)
#pragma unroll
      for (int c = 1; c < 4; ++c) {
        const int e = b * c;
        // w = exp(-/+ i 2 pi e / 16) = cos -/+ i sin
        const double2 w = make_double2(cs[e][0], INV ? cs[e][1] : -cs[e][1]);
        u[4 * c + b] = cmul(u[4 * c + b], w);
      }
    double2 y[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double2 t0 = u[4 * c], t1 = u[4 * c + 1], t2 = u[4 * c + 2], t3 = u[4 * c + 3];
      dft4<INV>(t0, t1, t2, t3);
      y[c] = t0;
      y[c + 4] = t1;
      y[c + 8] = t2;
      y[c + 12] = t3;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) u[q] = y[q];
  } else {  // R == 8: a_r = u_r + u_{r+4}, b_r = (u_r - u_{r+4}) w8^r, y_2q = DFT4(a), y_2q+1 = DFT4(b)
    const double h = 0.70710678118654752440;
    double2 a[4], b[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      a[r] = cadd(u[r], u[r + 4]);
      b[r] = csub(u[r], u[r + 4]);
    }
    // w8 = (1 - i)/sqrt2 (fwd), w8^2 = -i, w8^3 = (-1 - i)/sqrt2
    b[1] = INV ? make_double2(h * (b[1].x - b[1].y), h * (b[1].x + b[1].y))
               : make_double2(h * (b[1].x + b[1].y), h * (b[1].y - b[1].x));
    b[2] = rot<INV>(b[2]);
    b[3] = INV ? make_double2(-h * (b[3].x + b[3].y), h * (b[3].x - b[3].y))
               : make_double2(h * (b[3].y - b[3].x), -h * (b[3].x + b[3].y));
    dft4<INV>(a[0], a[1], a[2], a[3]);
    dft4<INV>(b[0], b[1], b[2], b[3]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      u[2 * q] = a[q];
      u[2 * q + 1] = b[q];
    }
  }
}

}  // namespace sdcsw
