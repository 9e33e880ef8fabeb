// Ring kernel: per (state, N/S ring pair) inverse longitude FFTs of the four
// synthesised fields, the pointwise nonlinear products on the Gaussian grid
// and the forward FFTs of the five products - all in shared memory, so grid
// data never touches HBM.  Replaces the irfft2 / products / rfft2 chain of the
// planar _f_expl (pkg/src/parsdc/problems/swe.py:176-185) with its spherical
// restatement (A=eta U, B=eta V, C=Phi' U, D=Phi' V,
// E=(U^2+V^2)/(2(1-mu^2))).
//
// FFT: mixed-radix (8, 4, 3) Stockham autosort over nlon = 3*2^k complex
// points (kernel templated on nlon: 96 ... 1536), in place: every pass reads all butterfly inputs of all the
// concurrent transforms into registers, synchronises, then writes.  The two
// real rings of a pair are packed into one complex transform (z = x_N + i x_S),
// and the 4 inverse / 5 forward transforms of a pair run as ONE multi-FFT each,
// so a pair costs 2 * (#radix passes) barrier phases instead of 9x that.
// Output per (b, pair, m <= T): the seven analysis data slots, pre-weighted,
// pre-multiplied by i m where the analysis needs it and folded into symmetric
// (N+S) / antisymmetric (N-S) parts.
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

// Shared-memory FFT arrays are padded by one element every 8: Stockham writes
// at stride R (and the radix-8 first pass in particular) then hit 8 distinct
// 16-byte bank groups per quarter-warp instead of one.
__device__ __forceinline__ int pz(int k) { return k + (k >> 3); }
template <int N>
constexpr int padded() { return N + N / 8; }

// Compile-time radix plan for nlon = 3 * 2^k: as many radix-8 passes as
// possible, then radix 4, then the radix-3 pass (p is a power of two before it).
constexpr int pow2_of(int n) { return n % 3 == 0 ? n / 3 : n; }
constexpr int log2i(int n) { return n <= 1 ? 0 : 1 + log2i(n / 2); }
constexpr int n8_of(int n) {
  return log2i(pow2_of(n)) % 3 == 1 ? log2i(pow2_of(n)) / 3 - 1 : log2i(pow2_of(n)) / 3;
}
constexpr int n4_of(int n) {
  return log2i(pow2_of(n)) % 3 == 1 ? 2 : (log2i(pow2_of(n)) % 3 == 2 ? 1 : 0);
}
constexpr int nstages_of(int n) { return n8_of(n) + n4_of(n) + (n % 3 == 0 ? 1 : 0); }
constexpr int radix_of(int n, int s) { return s < n8_of(n) ? 8 : (s < n8_of(n) + n4_of(n) ? 4 : 3); }

// One in-place Stockham pass (radix R, sub-length P) over NF concurrent
// transforms of length N stored at Z[f * N]; all index arithmetic is by
// compile-time constants.  tw[k] = exp(-2 pi i k / N) in shared memory.
template <int N, int R, int P, bool INV, int NF, int THREADS>
__device__ __forceinline__ void pass(double2* Z, const double2* tw) {
  constexpr int NR = N / R;
  constexpr int ITEMS = NF * NR;
  constexpr int TS = N / (R * P);
  constexpr int MAXIT = (ITEMS + THREADS - 1) / THREADS;
  double2 v[MAXIT][R];
#pragma unroll
  for (int q = 0; q < MAXIT; ++q) {
    const int it = threadIdx.x + q * THREADS;
    if (ITEMS % THREADS == 0 || it < ITEMS) {
      const int f = it / NR, i = it - f * NR;
      const double2* X = Z + f * padded<N>();
      const int k = i % P;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = X[pz(i + r * NR)];
      if (P > 1 && k) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = tw[r * k * TS];
          if (INV) w.y = -w.y;
          v[q][r] = cmul(v[q][r], w);
        }
      }
      dft<R, INV>(v[q]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < MAXIT; ++q) {
    const int it = threadIdx.x + q * THREADS;
    if (ITEMS % THREADS == 0 || it < ITEMS) {
      const int f = it / NR, i = it - f * NR;
      double2* X = Z + f * padded<N>();
      const int k = i % P;
      const int jo = (i - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) X[pz(jo + r * P)] = v[q][r];
    }
  }
  __syncthreads();
}

template <int N, int S, int P, bool INV, int NF, int THREADS>
__device__ __forceinline__ void passes(double2* Z, const double2* tw) {
  if constexpr (S < nstages_of(N)) {
    constexpr int R = radix_of(N, S);
    pass<N, R, P, INV, NF, THREADS>(Z, tw);
    passes<N, S + 1, P * R, INV, NF, THREADS>(Z, tw);
  }
}

template <int N, int THREADS>
__global__ void __launch_bounds__(THREADS) k_ring(const double2* __restrict__ fsyn,
                                                  double2* __restrict__ gan, int J, int T,
                                                  const double* __restrict__ mu,
                                                  const double* __restrict__ wsyn,
                                                  const double* __restrict__ wke,
                                                  const double2* __restrict__ twg,
                                                  double two_omega) {
  extern __shared__ double2 sm2[];
  const int L = T + 1;
  constexpr int NP = padded<N>();
  double2* Z = sm2;             // [5][NP] (padded)
  double2* tw = sm2 + 5 * NP;   // [N]
  const int j = blockIdx.x, b = blockIdx.y;
  const double2* F = fsyn + ((size_t)b * J + j) * L * 8;

  for (int k = threadIdx.x; k < N; k += THREADS) tw[k] = twg[k];
  // spectra of U, V, zeta, Phi:  Z_m = X_m + i Y_m,  Z_{N-m} = conj(X_m) + i conj(Y_m)
  for (int idx = threadIdx.x; idx < 4 * N; idx += THREADS) {
    const int k = idx >> 2, f = idx & 3;
    double2 z = make_double2(0.0, 0.0);
    if (k <= T) {
      double2 xn = F[(k * 4 + f) * 2], xs = F[(k * 4 + f) * 2 + 1];
      if (k == 0) xn.y = xs.y = 0.0;
      z = make_double2(xn.x - xs.y, xn.y + xs.x);
    } else if (k >= N - T) {
      const int m = N - k;
      const double2 xn = F[(m * 4 + f) * 2], xs = F[(m * 4 + f) * 2 + 1];
      z = make_double2(xn.x + xs.y, xs.x - xn.y);
    }
    Z[f * NP + pz(k)] = z;
  }
  __syncthreads();
  passes<N, 0, 1, true, 4, THREADS>(Z, tw);

  // products on the grid: re = north ring, im = south ring
  const double muj = mu[j];
  const double cor_n = two_omega * muj, cor_s = -two_omega * muj;
  const double ke_scale = 0.5 / ((1.0 - muj) * (1.0 + muj));
  for (int k0 = threadIdx.x; k0 < N; k0 += THREADS) {
    const int k = pz(k0);
    const double2 U = Z[k], V = Z[NP + k], Zt = Z[2 * NP + k], Ph = Z[3 * NP + k];
    const double en = Zt.x + cor_n, es = Zt.y + cor_s;
    Z[k] = make_double2(en * U.x, es * U.y);                       // A = eta U
    Z[NP + k] = make_double2(en * V.x, es * V.y);                  // B = eta V
    Z[2 * NP + k] = make_double2(Ph.x * U.x, Ph.y * U.y);          // C = Phi U
    Z[3 * NP + k] = make_double2(Ph.x * V.x, Ph.y * V.y);          // D = Phi V
    Z[4 * NP + k] = make_double2((U.x * U.x + V.x * V.x) * ke_scale,
                                (U.y * U.y + V.y * V.y) * ke_scale);  // kinetic energy
  }
  __syncthreads();
  passes<N, 0, 1, false, 5, THREADS>(Z, tw);

  const double ws = wsyn[j], wk = wke[j];
  const double h = 0.5 / (double)N;
  // analysis layout: [b][m][j][fold][slot]
  double2* out = gan + ((size_t)b * L * J + j) * (kNumSlots * 2);
  for (int idx = threadIdx.x; idx < 5 * L; idx += THREADS) {
    const int m = idx / 5, o = idx - 5 * m;
    const double2 zm = Z[o * NP + pz(m)], zc = Z[o * NP + pz(m == 0 ? 0 : N - m)];
    // X = FFT(north)/N, Y = FFT(south)/N; S = X + Y, A = X - Y
    const double2 X = make_double2(h * (zm.x + zc.x), h * (zm.y - zc.y));
    const double2 Y = make_double2(h * (zm.y + zc.y), -h * (zm.x - zc.x));
    const double2 S = cadd(X, Y), A = csub(X, Y);
    const double dm = (double)m;
    double2* dst = out + (size_t)m * J * (kNumSlots * 2);
    switch (o) {
      case 0:  // A = eta U:  X_zeta = -(i m A) ws,  Y_delta = A ws
        dst[0 * kNumSlots + kXZeta] = make_double2(dm * S.y * ws, -dm * S.x * ws);
        dst[1 * kNumSlots + kXZeta] = make_double2(dm * A.y * ws, -dm * A.x * ws);
        dst[0 * kNumSlots + kYDelta] = make_double2(S.x * ws, S.y * ws);
        dst[1 * kNumSlots + kYDelta] = make_double2(A.x * ws, A.y * ws);
        break;
      case 1:  // B = eta V:  X_delta = (i m B) ws,  Y_zeta = B ws
        dst[0 * kNumSlots + kXDelta] = make_double2(-dm * S.y * ws, dm * S.x * ws);
        dst[1 * kNumSlots + kXDelta] = make_double2(-dm * A.y * ws, dm * A.x * ws);
        dst[0 * kNumSlots + kYZeta] = make_double2(S.x * ws, S.y * ws);
        dst[1 * kNumSlots + kYZeta] = make_double2(A.x * ws, A.y * ws);
        break;
      case 2:  // C = Phi U:  X_phi = -(i m C) ws
        dst[0 * kNumSlots + kXPhi] = make_double2(dm * S.y * ws, -dm * S.x * ws);
        dst[1 * kNumSlots + kXPhi] = make_double2(dm * A.y * ws, -dm * A.x * ws);
        break;
      case 3:  // D = Phi V:  Y_phi = D ws
        dst[0 * kNumSlots + kYPhi] = make_double2(S.x * ws, S.y * ws);
        dst[1 * kNumSlots + kYPhi] = make_double2(A.x * ws, A.y * ws);
        break;
      default:  // kinetic energy: X_ke = E wk
        dst[0 * kNumSlots + kXKe] = make_double2(S.x * wk, S.y * wk);
        dst[1 * kNumSlots + kXKe] = make_double2(A.x * wk, A.y * wk);
        break;
    }
  }
}

#define SDCSW_RING_SIZES(X) X(96, 256) X(192, 256) X(384, 256) X(768, 256) X(1536, 512)

bool ring_supported(int nlon) {
#define SDCSW_RING_OK(NV, TV) if (nlon == NV) return true;
  SDCSW_RING_SIZES(SDCSW_RING_OK)
#undef SDCSW_RING_OK
  return false;
}

cudaError_t configure_ring(size_t smem) {
  cudaError_t e = cudaSuccess;
#define SDCSW_RING_CFG(NV, TV)                                                                     \
  if (e == cudaSuccess)                                                                            \
    e = cudaFuncSetAttribute(k_ring<NV, TV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  SDCSW_RING_SIZES(SDCSW_RING_CFG)
#undef SDCSW_RING_CFG
  return e;
}

size_t ring_smem_bytes(int nlon) { return (size_t)(5 * (nlon + nlon / 8) + nlon) * sizeof(double2); }

cudaError_t launch_ring(const Plan& p, int nb, cudaStream_t s) {
  dim3 grid(p.J, nb);
#define SDCSW_RING_LAUNCH(NV, TV)                                                                  \
  if (p.nlon == NV) {                                                                              \
    k_ring<NV, TV><<<grid, TV, p.ring_smem, s>>>(p.fsyn, p.gan, p.J, p.T, p.mu, p.wsyn, p.wke,      \
                                                 p.twiddle, 2.0 * p.omega);                        \
    return cudaGetLastError();                                                                     \
  }
  SDCSW_RING_SIZES(SDCSW_RING_LAUNCH)
#undef SDCSW_RING_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace sdcsw
