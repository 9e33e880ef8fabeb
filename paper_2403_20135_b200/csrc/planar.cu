// Planar doubly periodic shallow water: f_E on the GPU.
//
// Restates PlanarShallowWater._f_expl / _velocity
// (pkg/src/parsdc/problems/swe.py:174-205) for a batch of states:
//   psi = -zeta / k^2, chi = -delta / k^2, (u, v) = irfft2(-i ky psi + i kx chi,
//   i kx psi + i ky chi), q = f0 + irfft2(zeta), phi = irfft2(phi'),
//   flux = rfft2(q u, q v), kinetic = rfft2((u^2 + v^2) / 2), mass = rfft2(phi u, phi v),
//   (Phi'_t, zeta_t, delta_t) = (-(i kx mass_x + i ky mass_y), -(i kx flux_x + i ky flux_y),
//   (i kx flux_y - i ky flux_x) + k^2 kinetic) - nu k^4 state, times the 2/3 mask.
// Spectra are [N (kx)][NH = N/2 + 1 (ky)] (the reference's rfft2 layout).
//
// Three kernels per f_E, each a batch of shared-memory Stockham FFTs:
//   k_pcol_inv : per block of CW ky columns, the four fields U, V, zeta, Phi'
//                (velocity recovered in the load) -> inverse FFT along kx;
//   k_prow     : per block of RW grid rows, packed complex inverse FFTs (two
//                neighbouring rows of one field per transform; Hermitian
//                completion in the load), the five grid products, packed
//                forward FFTs, unpacked to the five row half-spectra;
//   k_pcol_fwd : per block of ky columns, five forward FFTs along kx and the
//                tendency assembly (derivatives, k^2 E, hyperviscosity, mask).
// The work buffers between them stay in L2 for the sizes the reference runs.
#include "fft_math.cuh"

namespace sdcsw {

template <int N> struct PPlan;
#define SDCSW_PPLAN(NV, NS, ...) \
  template <> struct PPlan<NV> { static constexpr int n = NS; static constexpr int r[4] = {__VA_ARGS__}; };
SDCSW_PPLAN(8, 1, 8)
SDCSW_PPLAN(12, 2, 4, 3)
SDCSW_PPLAN(16, 2, 4, 4)
SDCSW_PPLAN(24, 2, 8, 3)
SDCSW_PPLAN(32, 2, 8, 4)
SDCSW_PPLAN(48, 2, 16, 3)
SDCSW_PPLAN(64, 2, 8, 8)
SDCSW_PPLAN(96, 3, 8, 4, 3)
SDCSW_PPLAN(128, 2, 16, 8)
SDCSW_PPLAN(192, 3, 16, 4, 3)
SDCSW_PPLAN(256, 2, 16, 16)
SDCSW_PPLAN(384, 3, 16, 8, 3)
SDCSW_PPLAN(512, 3, 16, 8, 4)
SDCSW_PPLAN(768, 3, 16, 16, 3)
SDCSW_PPLAN(1024, 3, 16, 16, 4)
#undef SDCSW_PPLAN
#define SDCSW_PLANAR_SIZES(X) \
  X(8) X(12) X(16) X(24) X(32) X(48) X(64) X(96) X(128) X(192) X(256) X(384) X(512) X(768) X(1024)

constexpr int kPThreads = 256;
__device__ __forceinline__ int ppz(int k) { return k + (k >> 3); }
template <int N>
constexpr int ppad() { return N + N / 8; }
constexpr int pow2_floor(int x) {
  int p = 1;
  while (2 * p <= x) p *= 2;
  return p;
}
template <int N>
constexpr int col_width() {  // ky columns per column-kernel CTA
  const int w = pow2_floor(512 / N > 0 ? 512 / N : 1);
  return w > 8 ? 8 : w;
}
template <int N>
constexpr int row_count() {  // grid rows per row-kernel CTA (an even power of two dividing N)
  int w = pow2_floor(1024 / N > 2 ? 1024 / N : 2);
  w = w > 8 ? 8 : w;
  while (N % w) w /= 2;
  return w;
}
template <int N>
constexpr size_t col_smem(int nf) { return (size_t)(2 * nf * col_width<N>() * ppad<N>() + N) * 16; }
template <int N>
constexpr size_t row_smem() { return (size_t)(2 * 5 * (row_count<N>() / 2) * ppad<N>() + N) * 16; }

// One out-of-place Stockham pass (radix R, sub-length P) over NF transforms
// of length N; tw[k] = exp(-2 pi i k / N).
template <int N, int R, int P, bool INV, int NF>
__device__ __forceinline__ void ppass(const double2* __restrict__ in, double2* __restrict__ out,
                                      const double2* __restrict__ tw) {
  constexpr int NR = N / R;
  constexpr int TS = N / (R * P);
  constexpr int NPP = ppad<N>();
  for (int it = threadIdx.x; it < NF * NR; it += kPThreads) {
    const int f = it / NR, i = it - f * NR;
    const double2* X = in + f * NPP;
    double2* Y = out + f * NPP;
    const int k = i % P;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = X[ppz(i + r * NR)];
    if (P > 1 && k) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = tw[r * k * TS];
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    dft<R, INV>(v);
    const int jo = (i - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) Y[ppz(jo + r * P)] = v[r];
  }
  __syncthreads();
}
// All passes, ping-ponging a -> b -> a ...; the result is in a when the plan
// has an even number of passes, else in b.
template <int N, bool INV, int NF, int S = 0, int P = 1>
__device__ __forceinline__ void pfft(double2* a, double2* b, const double2* tw) {
  if constexpr (S < PPlan<N>::n) {
    constexpr int R = PPlan<N>::r[S];
    ppass<N, R, P, INV, NF>(a, b, tw);
    pfft<N, INV, NF, S + 1, P * R>(b, a, tw);
  }
}
template <int N>
__device__ __forceinline__ double2* pfft_result(double2* a, double2* b) {
  return PPlan<N>::n % 2 == 0 ? a : b;
}

// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(kPThreads) k_pcol_inv(const double2* __restrict__ u,
                                                        double2* __restrict__ w1,
                                                        const double* __restrict__ kx,
                                                        const double* __restrict__ ky,
                                                        const double* __restrict__ lam,
                                                        const double2* __restrict__ twg,
                                                        int* step_counter) {
  SDCSW_PDL_ENTRY();
  constexpr int CW = col_width<N>(), NH = N / 2 + 1, NPP = ppad<N>(), NF = 4 * CW;
  constexpr int C = N * NH;
  extern __shared__ double2 smp[];
  double2* A = smp;
  double2* B = A + NF * NPP;
  double2* tw = B + NF * NPP;
  for (int k = threadIdx.x; k < N; k += kPThreads) tw[k] = twg[k];
  SDCSW_PDL_WAIT();
  if (step_counter != nullptr && (blockIdx.x | blockIdx.y | threadIdx.x) == 0)
    atomicAdd(step_counter, 1);  // the stepper's step index (divergence reports)
  const int c0 = blockIdx.x * CW, b = blockIdx.y;
  const double2* st = u + (size_t)b * 3 * C;
  for (int e = threadIdx.x; e < N * CW; e += kPThreads) {
    const int kxi = e / CW, c = e - kxi * CW, kyi = c0 + c;
    double2 U = make_double2(0.0, 0.0), V = U, Z = U, F = U;
    if (kyi < NH) {
      const int idx = kxi * NH + kyi;
      F = st[idx];
      Z = st[C + idx];
      const double2 d = st[2 * C + idx];
      const double l = lam[idx];
      const double inv = l > 0.0 ? 1.0 / l : 0.0;
      const double2 psi = make_double2(-Z.x * inv, -Z.y * inv);
      const double2 chi = make_double2(-d.x * inv, -d.y * inv);
      const double a = kx[kxi], q = ky[kyi];
      // U = -i ky psi + i kx chi, V = i kx psi + i ky chi
      U = make_double2(q * psi.y - a * chi.y, a * chi.x - q * psi.x);
      V = make_double2(-a * psi.y - q * chi.y, a * psi.x + q * chi.x);
    }
    A[(0 * CW + c) * NPP + ppz(kxi)] = U;
    A[(1 * CW + c) * NPP + ppz(kxi)] = V;
    A[(2 * CW + c) * NPP + ppz(kxi)] = Z;
    A[(3 * CW + c) * NPP + ppz(kxi)] = F;
  }
  __syncthreads();
  pfft<N, true, NF>(A, B, tw);
  const double2* R = pfft_result<N>(A, B);
  for (int e = threadIdx.x; e < 4 * N * CW; e += kPThreads) {
    const int f = e / (N * CW), rem = e - f * N * CW, x = rem / CW, c = rem - x * CW;
    const int kyi = c0 + c;
    if (kyi < NH) w1[(((size_t)b * 4 + f) * N + x) * NH + kyi] = R[(f * CW + c) * NPP + ppz(x)];
  }
}

// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(kPThreads) k_prow(const double2* __restrict__ w1,
                                                    double2* __restrict__ w2,
                                                    const double2* __restrict__ twg, double f0) {
  SDCSW_PDL_ENTRY();
  constexpr int RW = row_count<N>(), NH = N / 2 + 1, NPP = ppad<N>(), H = N / 2;
  constexpr int RP = RW / 2;  // row pairs: rows 2p (real part) and 2p + 1 (imaginary part)
  extern __shared__ double2 smp[];
  double2* A = smp;
  double2* B = A + 5 * RP * NPP;
  double2* tw = B + 5 * RP * NPP;
  for (int k = threadIdx.x; k < N; k += kPThreads) tw[k] = twg[k];
  SDCSW_PDL_WAIT();
  const int x0 = blockIdx.x * RW, b = blockIdx.y;
  // transform t = f RP + p packs rows x0 + 2p, x0 + 2p + 1 of field f (U, V, zeta,
  // Phi'): one field, neighbouring rows - similar magnitudes, so sharing one
  // complex FFT costs no relative accuracy.  Hermitian completion per row:
  // Z[k] = X[k] + i Y[k], Z[N-k] = conj(X[k]) + i conj(Y[k]); the imaginary
  // parts of the k = 0 and k = N/2 terms are ignored (as irfft does).
  for (int e = threadIdx.x; e < 4 * RP * N; e += kPThreads) {
    const int t = e / N, k = e - t * N, f = t / RP, pr = t - f * RP;
    const int kk = k <= H ? k : N - k;
    const double2* row = w1 + (((size_t)b * 4 + f) * N + x0 + 2 * pr) * NH;
    double2 X = row[kk], Y = row[NH + kk];
    if (kk == 0 || kk == H) X.y = Y.y = 0.0;
    A[t * NPP + ppz(k)] =
        k <= H ? make_double2(X.x - Y.y, X.y + Y.x) : make_double2(X.x + Y.y, Y.x - X.y);
  }
  __syncthreads();
  pfft<N, true, 4 * RP>(A, B, tw);
  double2* R1 = pfft_result<N>(A, B);
  double2* O = R1 == A ? B : A;
  const double s = 1.0 / ((double)N * (double)N);  // irfft2 normalisation
  for (int e = threadIdx.x; e < RP * N; e += kPThreads) {
    const int pr = e / N, n = e - pr * N;
    const double2 zu = R1[(0 * RP + pr) * NPP + ppz(n)], zv = R1[(1 * RP + pr) * NPP + ppz(n)];
    const double2 zz = R1[(2 * RP + pr) * NPP + ppz(n)], zp = R1[(3 * RP + pr) * NPP + ppz(n)];
    double2 o[5];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // h = 0: row 2p (real parts), 1: row 2p + 1
      const double uu = (h ? zu.y : zu.x) * s, vv = (h ? zv.y : zv.x) * s;
      const double zeta = (h ? zz.y : zz.x) * s, phi = (h ? zp.y : zp.x) * s;
      const double q = f0 + zeta;
      const double val[5] = {q * uu, q * vv, 0.5 * (uu * uu + vv * vv), phi * uu, phi * vv};
#pragma unroll
      for (int f = 0; f < 5; ++f) {
        if (h) o[f].y = val[f];
        else o[f].x = val[f];
      }
    }
    // products (q u, q v, kinetic, Phi' u, Phi' v), row pairs packed again
#pragma unroll
    for (int f = 0; f < 5; ++f) O[(f * RP + pr) * NPP + ppz(n)] = o[f];
  }
  __syncthreads();
  pfft<N, false, 5 * RP>(O, R1, tw);
  const double2* R2 = pfft_result<N>(O, R1);
  // unpack: F(row 2p)[k] = (P[k] + conj(P[N-k])) / 2, F(row 2p+1)[k] = (P[k] - conj(P[N-k])) / 2i
  for (int e = threadIdx.x; e < 5 * RP * NH; e += kPThreads) {
    const int t = e / NH, k = e - t * NH, f = t / RP, pr = t - f * RP, kc = k == 0 ? 0 : N - k;
    const double2 a = R2[t * NPP + ppz(k)], c = R2[t * NPP + ppz(kc)];
    double2* dst = w2 + (((size_t)b * 5 + f) * N + x0 + 2 * pr) * NH + k;
    dst[0] = make_double2(0.5 * (a.x + c.x), 0.5 * (a.y - c.y));
    dst[NH] = make_double2(0.5 * (a.y + c.y), -0.5 * (a.x - c.x));
  }
}

// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(kPThreads) k_pcol_fwd(const double2* __restrict__ w2,
                                                        const double2* __restrict__ u,
                                                        double2* __restrict__ fe,
                                                        const double* __restrict__ kx,
                                                        const double* __restrict__ ky,
                                                        const double* __restrict__ lam,
                                                        const double2* __restrict__ twg,
                                                        double nu) {
  SDCSW_PDL_ENTRY();
  constexpr int CW = col_width<N>(), NH = N / 2 + 1, NPP = ppad<N>(), NF = 5 * CW;
  constexpr int C = N * NH, KEEP = (N - 1) / 3;
  extern __shared__ double2 smp[];
  double2* A = smp;
  double2* B = A + NF * NPP;
  double2* tw = B + NF * NPP;
  for (int k = threadIdx.x; k < N; k += kPThreads) tw[k] = twg[k];
  SDCSW_PDL_WAIT();
  const int c0 = blockIdx.x * CW, b = blockIdx.y;
  for (int e = threadIdx.x; e < 5 * N * CW; e += kPThreads) {
    const int f = e / (N * CW), rem = e - f * N * CW, x = rem / CW, c = rem - x * CW;
    const int kyi = c0 + c;
    A[(f * CW + c) * NPP + ppz(x)] =
        kyi < NH ? w2[(((size_t)b * 5 + f) * N + x) * NH + kyi] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  pfft<N, false, NF>(A, B, tw);
  const double2* R = pfft_result<N>(A, B);
  const double2* st = u + (size_t)b * 3 * C;
  double2* out = fe + (size_t)b * 3 * C;
  for (int e = threadIdx.x; e < N * CW; e += kPThreads) {
    const int kxi = e / CW, c = e - kxi * CW, kyi = c0 + c;
    if (kyi >= NH) continue;
    const int idx = kxi * NH + kyi;
    const int ix = kxi < N / 2 ? kxi : kxi - N;
    const bool keep = (ix < 0 ? -ix : ix) <= KEEP && kyi <= KEEP;
    double2 t0 = make_double2(0.0, 0.0), t1 = t0, t2 = t0;
    if (keep) {
      const double2 fx = R[(0 * CW + c) * NPP + ppz(kxi)], fy = R[(1 * CW + c) * NPP + ppz(kxi)];
      const double2 ke = R[(2 * CW + c) * NPP + ppz(kxi)];
      const double2 mx = R[(3 * CW + c) * NPP + ppz(kxi)], my = R[(4 * CW + c) * NPP + ppz(kxi)];
      const double a = kx[kxi], q = ky[kyi], l = lam[idx];
      // i k z = (-k z.y, k z.x)
      t0 = make_double2(a * mx.y + q * my.y, -(a * mx.x + q * my.x));
      t1 = make_double2(a * fx.y + q * fy.y, -(a * fx.x + q * fy.x));
      t2 = make_double2((q * fx.y - a * fy.y) + l * ke.x, (a * fy.x - q * fx.x) + l * ke.y);
      if (nu > 0.0) {
        const double h = nu * (l * l);
        const double2 s0 = st[idx], s1 = st[C + idx], s2 = st[2 * C + idx];
        t0 = make_double2(t0.x - h * s0.x, t0.y - h * s0.y);
        t1 = make_double2(t1.x - h * s1.x, t1.y - h * s1.y);
        t2 = make_double2(t2.x - h * s2.x, t2.y - h * s2.y);
      }
    }
    out[idx] = t0;
    out[C + idx] = t1;
    out[2 * C + idx] = t2;
  }
}

bool planar_supported(int n) {
#define SDCSW_P_OK(NV) if (n == NV) return true;
  SDCSW_PLANAR_SIZES(SDCSW_P_OK)
#undef SDCSW_P_OK
  return false;
}

cudaError_t configure_planar(int n) {
  cudaError_t e = cudaSuccess;
#define SDCSW_P_CFG(NV)                                                                          \
  if (n == NV) {                                                                                 \
    e = cudaFuncSetAttribute(k_pcol_inv<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                             (int)col_smem<NV>(4));                                              \
    if (e == cudaSuccess)                                                                        \
      e = cudaFuncSetAttribute(k_prow<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                               (int)row_smem<NV>());                                             \
    if (e == cudaSuccess)                                                                        \
      e = cudaFuncSetAttribute(k_pcol_fwd<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                               (int)col_smem<NV>(5));                                            \
    return e;                                                                                    \
  }
  SDCSW_PLANAR_SIZES(SDCSW_P_CFG)
#undef SDCSW_P_CFG
  return cudaErrorInvalidValue;
}

cudaError_t planar_f_expl(const Plan& p, const double2* u, double2* fe, int nb, cudaStream_t s,
                          int* step_counter) {
#define SDCSW_P_RUN(NV)                                                                           \
  if (p.pn == NV) {                                                                               \
    constexpr int NH = NV / 2 + 1;                                                                \
    const dim3 gc((NH + col_width<NV>() - 1) / col_width<NV>(), nb);                              \
    launch_k(k_pcol_inv<NV>, gc, kPThreads, col_smem<NV>(4), s, u, p.pw1, p.pkx, p.pky, p.lam,    \
             p.ptw, step_counter);                                                                \
    launch_k(k_prow<NV>, dim3(NV / row_count<NV>(), nb), kPThreads, row_smem<NV>(), s,            \
             (const double2*)p.pw1, p.pw2, p.ptw, p.pf0);                                         \
    launch_k(k_pcol_fwd<NV>, gc, kPThreads, col_smem<NV>(5), s, (const double2*)p.pw2, u, fe,     \
             p.pkx, p.pky, p.lam, p.ptw, p.pnu);                                                  \
    return cudaGetLastError();                                                                    \
  }
  SDCSW_PLANAR_SIZES(SDCSW_P_RUN)
#undef SDCSW_P_RUN
  return cudaErrorInvalidValue;
}

}  // namespace sdcsw
