// Ring kernel: per (state, N/S ring pair) inverse longitude FFTs of the four
// synthesised fields, the pointwise nonlinear products on the Gaussian grid
// and the forward FFTs of the five products - all in shared memory, so grid
// data never touches HBM.  Replaces the irfft2 / products / rfft2 chain of the
// planar _f_expl (pkg/src/parsdc/problems/swe.py:176-185) with its spherical
// restatement (A=eta U, B=eta V, C=Phi' U, D=Phi' V,
// E=(U^2+V^2)/(2(1-mu^2))).
//
// FFT: mixed-radix (4, 2, 3) Stockham autosort over nlon = 2^k or 3*2^k
// complex points; two real rings (north, south) are packed into one complex
// transform (z = x_N + i x_S), so 4 inverse + 5 forward complex FFTs of length
// nlon per ring pair.  Output per (b, pair, m <= T): the seven analysis data
// slots, pre-weighted, pre-multiplied by i m where the analysis needs it and
// folded into symmetric (N+S) / antisymmetric (N-S) parts.
#include "internal.cuh"

namespace sdcsw {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// in-place-ish Stockham: ping-pong between x and y; returns the buffer holding
// the result.  Ends with __syncthreads().
template <bool INV>
__device__ double2* fft_stockham(double2* x, double2* y, const FftPlan& fp,
                                 const double2* __restrict__ tw) {
  const int N = fp.n;
  int p = 1;
  for (int st = 0; st < fp.nstages; ++st) {
    const int R = fp.radix[st];
    const int NR = N / R;
    const int ts = N / (R * p);
    for (int i = threadIdx.x; i < NR; i += blockDim.x) {
      const int k = i % p;
      const int jo = (i - k) * R + k;
      if (R == 4) {
        double2 u0 = x[i], u1 = x[i + NR], u2 = x[i + 2 * NR], u3 = x[i + 3 * NR];
        if (k) {
          double2 w1 = __ldg(tw + k * ts), w2 = __ldg(tw + 2 * k * ts), w3 = __ldg(tw + 3 * k * ts);
          if (INV) { w1.y = -w1.y; w2.y = -w2.y; w3.y = -w3.y; }
          u1 = cmul(u1, w1); u2 = cmul(u2, w2); u3 = cmul(u3, w3);
        }
        const double2 a0 = make_double2(u0.x + u2.x, u0.y + u2.y);
        const double2 a1 = make_double2(u0.x - u2.x, u0.y - u2.y);
        const double2 a2 = make_double2(u1.x + u3.x, u1.y + u3.y);
        const double2 a3 = make_double2(u1.x - u3.x, u1.y - u3.y);
        // forward: y1 = a1 - i a3, y3 = a1 + i a3 ; inverse swaps
        const double2 ia3 = INV ? make_double2(-a3.y, a3.x) : make_double2(a3.y, -a3.x);
        y[jo] = make_double2(a0.x + a2.x, a0.y + a2.y);
        y[jo + p] = make_double2(a1.x + ia3.x, a1.y + ia3.y);
        y[jo + 2 * p] = make_double2(a0.x - a2.x, a0.y - a2.y);
        y[jo + 3 * p] = make_double2(a1.x - ia3.x, a1.y - ia3.y);
      } else if (R == 2) {
        double2 u0 = x[i], u1 = x[i + NR];
        if (k) {
          double2 w1 = __ldg(tw + k * ts);
          if (INV) w1.y = -w1.y;
          u1 = cmul(u1, w1);
        }
        y[jo] = make_double2(u0.x + u1.x, u0.y + u1.y);
        y[jo + p] = make_double2(u0.x - u1.x, u0.y - u1.y);
      } else {  // R == 3
        double2 u0 = x[i], u1 = x[i + NR], u2 = x[i + 2 * NR];
        if (k) {
          double2 w1 = __ldg(tw + k * ts), w2 = __ldg(tw + 2 * k * ts);
          if (INV) { w1.y = -w1.y; w2.y = -w2.y; }
          u1 = cmul(u1, w1); u2 = cmul(u2, w2);
        }
        const double s3 = 0.86602540378443864676;  // sqrt(3)/2
        const double2 t1 = make_double2(u1.x + u2.x, u1.y + u2.y);
        const double2 t2 = make_double2(u0.x - 0.5 * t1.x, u0.y - 0.5 * t1.y);
        const double2 d = make_double2(u1.x - u2.x, u1.y - u2.y);
        // forward: y1 = t2 - i s d, y2 = t2 + i s d ; inverse swaps
        const double2 isd = INV ? make_double2(-s3 * d.y, s3 * d.x) : make_double2(s3 * d.y, -s3 * d.x);
        y[jo] = make_double2(u0.x + t1.x, u0.y + t1.y);
        y[jo + p] = make_double2(t2.x + isd.x, t2.y + isd.y);
        y[jo + 2 * p] = make_double2(t2.x - isd.x, t2.y - isd.y);
      }
    }
    __syncthreads();
    double2* tmp = x; x = y; y = tmp;
    p *= R;
  }
  return x;
}

__global__ void __launch_bounds__(256) k_ring(const double2* __restrict__ fsyn,
                                              double2* __restrict__ gan, int J, int T,
                                              const double* __restrict__ mu,
                                              const double* __restrict__ wsyn,
                                              const double* __restrict__ wke,
                                              const double2* __restrict__ tw, FftPlan fp,
                                              double two_omega) {
  extern __shared__ double2 sm2[];
  const int N = fp.n;
  const int L = T + 1;
  double2* buf0 = sm2;
  double2* buf1 = sm2 + N;
  double* grid = reinterpret_cast<double*>(sm2 + 2 * N);  // [4 fields][2 rings][N]
  const int j = blockIdx.x, b = blockIdx.y;
  const double2* F = fsyn + ((size_t)b * J + j) * L * 8;

  // ---- inverse transforms: U, V, zeta, Phi (north + i south) ----
  for (int f = 0; f < 4; ++f) {
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      double2 z = make_double2(0.0, 0.0);
      if (k <= T) {
        double2 xn = F[(k * 4 + f) * 2], xs = F[(k * 4 + f) * 2 + 1];
        if (k == 0) xn.y = xs.y = 0.0;
        z = make_double2(xn.x - xs.y, xn.y + xs.x);  // X + i Y
      } else if (k >= N - T) {
        const int m = N - k;
        const double2 xn = F[(m * 4 + f) * 2], xs = F[(m * 4 + f) * 2 + 1];
        z = make_double2(xn.x + xs.y, xs.x - xn.y);  // conj(X) + i conj(Y)
      }
      buf0[k] = z;
    }
    __syncthreads();
    const double2* res = fft_stockham<true>(buf0, buf1, fp, tw);
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      const double2 z = res[k];
      grid[(2 * f) * N + k] = z.x;
      grid[(2 * f + 1) * N + k] = z.y;
    }
    __syncthreads();
  }

  // ---- products and forward transforms ----
  const double muj = mu[j];
  const double cor_n = two_omega * muj, cor_s = -two_omega * muj;
  const double ke_scale = 0.5 / ((1.0 - muj) * (1.0 + muj));
  const double ws = wsyn[j], wk = wke[j];
  const double invn = 1.0 / (double)N;
  double2* out = gan + ((size_t)b * J + j) * L * (kNumSlots * 2);
  for (int o = 0; o < 5; ++o) {
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      double v[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double U = grid[(0 + s) * N + k], V = grid[(2 + s) * N + k];
        const double Z = grid[(4 + s) * N + k], Ph = grid[(6 + s) * N + k];
        const double eta = Z + (s ? cor_s : cor_n);
        switch (o) {
          case 0: v[s] = eta * U; break;
          case 1: v[s] = eta * V; break;
          case 2: v[s] = Ph * U; break;
          case 3: v[s] = Ph * V; break;
          default: v[s] = (U * U + V * V) * ke_scale; break;
        }
      }
      buf0[k] = make_double2(v[0], v[1]);
    }
    __syncthreads();
    const double2* res = fft_stockham<false>(buf0, buf1, fp, tw);
    for (int m = threadIdx.x; m <= T; m += blockDim.x) {
      const double2 zm = res[m], zc = res[m == 0 ? 0 : N - m];
      // X = FFT(north)/N, Y = FFT(south)/N
      const double2 X = make_double2(0.5 * (zm.x + zc.x) * invn, 0.5 * (zm.y - zc.y) * invn);
      const double2 Y = make_double2(0.5 * (zm.y + zc.y) * invn, -0.5 * (zm.x - zc.x) * invn);
      const double2 S = make_double2(X.x + Y.x, X.y + Y.y);   // symmetric fold
      const double2 A = make_double2(X.x - Y.x, X.y - Y.y);   // antisymmetric fold
      const double dm = (double)m;
      double2* dst = out + (size_t)m * (kNumSlots * 2);
      // i m z = (-m z.y, m z.x)
      switch (o) {
        case 0:  // A = eta U:  X_zeta = -(i m A) ws,  Y_delta = A ws
          dst[kXZeta * 2 + 0] = make_double2(dm * S.y * ws, -dm * S.x * ws);
          dst[kXZeta * 2 + 1] = make_double2(dm * A.y * ws, -dm * A.x * ws);
          dst[kYDelta * 2 + 0] = make_double2(S.x * ws, S.y * ws);
          dst[kYDelta * 2 + 1] = make_double2(A.x * ws, A.y * ws);
          break;
        case 1:  // B = eta V:  X_delta = (i m B) ws,  Y_zeta = B ws
          dst[kXDelta * 2 + 0] = make_double2(-dm * S.y * ws, dm * S.x * ws);
          dst[kXDelta * 2 + 1] = make_double2(-dm * A.y * ws, dm * A.x * ws);
          dst[kYZeta * 2 + 0] = make_double2(S.x * ws, S.y * ws);
          dst[kYZeta * 2 + 1] = make_double2(A.x * ws, A.y * ws);
          break;
        case 2:  // C = Phi U:  X_phi = -(i m C) ws
          dst[kXPhi * 2 + 0] = make_double2(dm * S.y * ws, -dm * S.x * ws);
          dst[kXPhi * 2 + 1] = make_double2(dm * A.y * ws, -dm * A.x * ws);
          break;
        case 3:  // D = Phi V:  Y_phi = D ws
          dst[kYPhi * 2 + 0] = make_double2(S.x * ws, S.y * ws);
          dst[kYPhi * 2 + 1] = make_double2(A.x * ws, A.y * ws);
          break;
        default:  // kinetic energy: X_ke = E wk
          dst[kXKe * 2 + 0] = make_double2(S.x * wk, S.y * wk);
          dst[kXKe * 2 + 1] = make_double2(A.x * wk, A.y * wk);
          break;
      }
    }
    __syncthreads();
  }
}

cudaError_t configure_ring(size_t smem) {
  return cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_ring(const Plan& p, int nb, cudaStream_t s) {
  dim3 grid(p.J, nb);
  k_ring<<<grid, p.ring_threads, p.ring_smem, s>>>(p.fsyn, p.gan, p.J, p.T, p.mu, p.wsyn, p.wke,
                                                   p.twiddle, p.fft, 2.0 * p.omega);
  return cudaGetLastError();
}

}  // namespace sdcsw
