// Legendre synthesis / analysis as grouped FP64 tensor-core GEMMs (DMMA).
//
// Per zonal wavenumber m the transforms are small dense GEMMs between the
// parity-sorted Legendre tables (rows = degree n, columns = northern
// latitudes j) and the batch of spectral coefficients / folded Fourier
// coefficients.  sm_100a has no tcgen05 kind for f64, so the tensor-core path
// is warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  The table - the large
// streamed operand - is read straight from HBM/L2 into A fragments; the small
// per-m coefficient slice is staged in shared memory and read as B fragments.
//
// Synthesis (replaces the inverse transforms inside the
// planar _f_expl, pkg/src/parsdc/problems/swe.py:176-178, 200-205):
//   E[j,c] = sum_{n-m even} P X + sum_{n-m odd} H Y,  O[j,c] = other parities,
//   north = E + O, south = E - O;  X/Y per column (U, V, zeta, Phi).
// Analysis (replaces the forward transforms, swe.py:180-190):
//   out[n,c] = sum_j P[n,j] Xfold[j,c] + sum_j H[n,j] Yfold[j,c]
//   with the fold (N+S or N-S) chosen by the parity class of row n.
#include "internal.cuh"

namespace sdcsw {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// synthesis: u [nb][3][C] -> fsyn [nb][J][L][4 (U,V,zeta,Phi)][2 (N,S)]
// grid (T+1, J / (16 warps), ceil(nb / NB)), block 32*warps
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(128) k_synthesis(
    const double2* __restrict__ u, int nb, int T, int J, int C, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, const int* __restrict__ row_n, const int* __restrict__ moff,
    const double* __restrict__ inv_nn, double radius, double2* __restrict__ fsyn,
    int* step_counter) {
  constexpr int PC = 8 * NB;        // P columns: (U,V) of all b, then (zeta,Phi) of all b
  constexpr int TH = (NB + 1) / 2;  // H tiles (U,V columns only)
  constexpr int HC = 8 * TH;
  constexpr int PS = PC + 4;        // strides = 4 or 12 (mod 16): conflict-free B fragments
  constexpr int HS = HC + 4;
  __shared__ double xp[kSynthChunk * PS];
  __shared__ double xh[kSynthChunk * HS];

  const int m = blockIdx.x;
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int j0 = (blockIdx.y * warps + warp) * kRowsPerWarp;
  const int b0 = blockIdx.z * NB;
  const int L = T + 1;
  if (step_counter != nullptr && (blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) == 0)
    atomicAdd(step_counter, 1);

  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  const int mo = moff[m];
  const double* P = ptab + (size_t)r0m * J + j0 + g;
  const double* H = htab + (size_t)r0m * J + j0 + g;
  const double dm = (double)m;

  double accE[2][NB][2], accO[2][NB][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) accE[a][c][0] = accE[a][c][1] = accO[a][c][0] = accO[a][c][1] = 0.0;

  for (int c0 = 0; c0 < rows; c0 += kSynthChunk) {
    const int nr = min(kSynthChunk, rows - c0);
    __syncthreads();
    // stage X (P data) and Y (H data) for rows [c0, c0+nr), batch columns
    for (int it = threadIdx.x; it < kSynthChunk * 2 * TH; it += blockDim.x) {
      const int rr = it / (2 * TH), b = it % (2 * TH);
      double2 uu = {0, 0}, vv = {0, 0}, zz = {0, 0}, pp = {0, 0}, uh = {0, 0}, vh = {0, 0};
      const int n = rr < nr ? row_n[r0m + c0 + rr] : -1;
      if (n >= 0 && b < NB && b0 + b < nb) {
        const int idx = mo + n - m;
        const double2* s = u + (size_t)(b0 + b) * 3 * C;
        const double2 phi = s[idx], zeta = s[C + idx], delta = s[2 * C + idx];
        const double il = inv_nn[idx];
        const double sm = dm * radius * il;  // i m chi / a = -i m a il delta
        const double sa = radius * il;
        uu = make_double2(sm * delta.y, -sm * delta.x);
        vv = make_double2(sm * zeta.y, -sm * zeta.x);
        zz = zeta;
        pp = phi;
        uh = make_double2(sa * zeta.x, sa * zeta.y);     // -psi / a
        vh = make_double2(-sa * delta.x, -sa * delta.y);  // chi / a
      }
      double* rp = xp + rr * PS;
      double* rh = xh + rr * HS;
      if (b < NB) {
        rp[4 * b + 0] = uu.x; rp[4 * b + 1] = uu.y; rp[4 * b + 2] = vv.x; rp[4 * b + 3] = vv.y;
        rp[4 * NB + 4 * b + 0] = zz.x; rp[4 * NB + 4 * b + 1] = zz.y;
        rp[4 * NB + 4 * b + 2] = pp.x; rp[4 * NB + 4 * b + 3] = pp.y;
      }
      rh[4 * b + 0] = uh.x; rh[4 * b + 1] = uh.y; rh[4 * b + 2] = vh.x; rh[4 * b + 3] = vh.y;
    }
    __syncthreads();
    if (j0 < J) {
      const int nsteps = nr >> 2;
      for (int s = 0; s < nsteps; ++s) {
        const int r = c0 + 4 * s;
        const size_t off = (size_t)(r + t) * J;
        double aP[2], aH[2];
        aP[0] = __ldg(P + off);
        aP[1] = __ldg(P + off + 8);
        aH[0] = __ldg(H + off);
        aH[1] = __ldg(H + off + 8);
        double bP[NB], bH[TH];
#pragma unroll
        for (int c = 0; c < NB; ++c) bP[c] = xp[(4 * s + t) * PS + 8 * c + g];
#pragma unroll
        for (int c = 0; c < TH; ++c) bH[c] = xh[(4 * s + t) * HS + 8 * c + g];
        if (r < le) {
#pragma unroll
          for (int a = 0; a < 2; ++a) {
#pragma unroll
            for (int c = 0; c < NB; ++c) dmma(accE[a][c], aP[a], bP[c]);
#pragma unroll
            for (int c = 0; c < TH; ++c) dmma(accO[a][c], aH[a], bH[c]);
          }
        } else {
#pragma unroll
          for (int a = 0; a < 2; ++a) {
#pragma unroll
            for (int c = 0; c < NB; ++c) dmma(accO[a][c], aP[a], bP[c]);
#pragma unroll
            for (int c = 0; c < TH; ++c) dmma(accE[a][c], aH[a], bH[c]);
          }
        }
      }
    }
  }
  if (j0 >= J) return;
  // epilogue: thread holds (re, im) of column pair 8c + 2t at rows j0 + 8a + g
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const int col = 8 * c + 2 * t;
    int b, f;
    if (col < 4 * NB) {
      b = col >> 2;
      f = (col & 3) >> 1;  // 0 = U, 1 = V
    } else {
      b = (col - 4 * NB) >> 2;
      f = 2 + (((col - 4 * NB) & 3) >> 1);  // 2 = zeta, 3 = Phi
    }
    if (b0 + b >= nb) continue;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int j = j0 + 8 * a + g;
      double2* dst = fsyn + ((((size_t)(b0 + b) * J + j) * L + m) * 4 + f) * 2;
      dst[0] = make_double2(accE[a][c][0] + accO[a][c][0], accE[a][c][1] + accO[a][c][1]);
      dst[1] = make_double2(accE[a][c][0] - accO[a][c][0], accE[a][c][1] - accO[a][c][1]);
    }
  }
}

// ---------------------------------------------------------------------------
// analysis: gan [nb][J][L][7][2 (S,A)] -> fe [nb][3][C]
// grid (n_work, ceil(nb / NB)), block 32*warps; work = (m << 16) | row block
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(128) k_analysis(
    const double2* __restrict__ gan, int nb, int T, int J, int C, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, const int* __restrict__ row_n, const int* __restrict__ moff,
    const double* __restrict__ lam, const int* __restrict__ work, double2* __restrict__ fe) {
  constexpr int PC = 8 * NB;        // (phi, zeta, delta) of all b, then ke of all b
  constexpr int HU = 6 * NB;        // H columns actually used
  constexpr int TH = (HU + 7) / 8;
  constexpr int HC = 8 * TH;
  constexpr int PS = PC + 4;
  constexpr int HS = HC + 4;
  constexpr int OS = PC + 1;
  __shared__ double dp[2][kAnalChunk * PS];
  __shared__ double dh[2][kAnalChunk * HS];
  static_assert(4 * kRowsPerWarp * OS <= 2 * kAnalChunk * PS, "output tile aliases dp");

  const int wk = work[blockIdx.x];
  const int m = wk >> 16, rb = wk & 0xffff;
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int b0 = blockIdx.y * NB;
  const int L = T + 1;
  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  const int rw = (rb * warps + warp) * kRowsPerWarp;
  const bool active = rw < rows;
  const bool ev0 = rw < le, ev1 = rw + 8 < le;
  const double* P = ptab + (size_t)(r0m + rw + g) * J + t;
  const double* H = htab + (size_t)(r0m + rw + g) * J + t;

  double acc[2][NB][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;

  for (int jc = 0; jc < J; jc += kAnalChunk) {
    const int nj = min(kAnalChunk, J - jc);
    __syncthreads();
    for (int it = threadIdx.x; it < kAnalChunk * NB; it += blockDim.x) {
      const int jj = it / NB, b = it % NB;
      double2 v[kNumSlots][2];
      if (jj < nj && b0 + b < nb) {
        const double2* src = gan + (((size_t)(b0 + b) * J + jc + jj) * L + m) * (kNumSlots * 2);
#pragma unroll
        for (int q = 0; q < kNumSlots * 2; ++q) v[q >> 1][q & 1] = src[q];
      } else {
#pragma unroll
        for (int q = 0; q < kNumSlots * 2; ++q) v[q >> 1][q & 1] = make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        double* rp = dp[f] + jj * PS;
        double* rh = dh[f] + jj * HS;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          rp[6 * b + 2 * q] = v[kXPhi + q][f].x;
          rp[6 * b + 2 * q + 1] = v[kXPhi + q][f].y;
          rh[6 * b + 2 * q] = v[kYPhi + q][f].x;
          rh[6 * b + 2 * q + 1] = v[kYPhi + q][f].y;
        }
        rp[6 * NB + 2 * b] = v[kXKe][f].x;
        rp[6 * NB + 2 * b + 1] = v[kXKe][f].y;
        if (b == 0)
          for (int q = HU; q < HC; ++q) rh[q] = 0.0;
      }
    }
    __syncthreads();
    if (active) {
      const int nsteps = nj >> 2;
      for (int s = 0; s < nsteps; ++s) {
        const int k = jc + 4 * s;
        double aP[2], aH[2];
        aP[0] = __ldg(P + k);
        aP[1] = __ldg(P + k + 8 * (size_t)J);
        aH[0] = __ldg(H + k);
        aH[1] = __ldg(H + k + 8 * (size_t)J);
        const int sr = (4 * s + t);
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          const double bs = dp[0][sr * PS + 8 * c + g];
          const double ba = dp[1][sr * PS + 8 * c + g];
          dmma(acc[0][c], aP[0], ev0 ? bs : ba);
          dmma(acc[1][c], aP[1], ev1 ? bs : ba);
        }
#pragma unroll
        for (int c = 0; c < TH; ++c) {
          const double bs = dh[0][sr * HS + 8 * c + g];
          const double ba = dh[1][sr * HS + 8 * c + g];
          dmma(acc[0][c], aH[0], ev0 ? ba : bs);
          dmma(acc[1][c], aH[1], ev1 ? ba : bs);
        }
      }
    }
  }
  __syncthreads();  // the output tiles alias dp
  if (!active) return;
  double* o = &dp[0][0] + warp * kRowsPerWarp * OS;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      o[(8 * a + g) * OS + 8 * c + 2 * t] = acc[a][c][0];
      o[(8 * a + g) * OS + 8 * c + 2 * t + 1] = acc[a][c][1];
    }
  __syncwarp();
  const int mo = moff[m];
  for (int it = lane; it < kRowsPerWarp * NB; it += 32) {
    const int rr = it % kRowsPerWarp, b = it / kRowsPerWarp;
    if (rw + rr >= rows || b0 + b >= nb) continue;
    const int n = row_n[r0m + rw + rr];
    if (n < 0) continue;
    const int idx = mo + n - m;
    const double* row = o + rr * OS;
    const double l = lam[idx];
    double2 phi = make_double2(row[6 * b + 0], row[6 * b + 1]);
    double2 zeta = make_double2(row[6 * b + 2], row[6 * b + 3]);
    double2 delta = make_double2(row[6 * b + 4] + l * row[6 * NB + 2 * b],
                                 row[6 * b + 5] + l * row[6 * NB + 2 * b + 1]);
    if (m == 0) phi.y = zeta.y = delta.y = 0.0;
    double2* dst = fe + (size_t)(b0 + b) * 3 * C;
    dst[idx] = phi;
    dst[C + idx] = zeta;
    dst[2 * C + idx] = delta;
  }
}

static int pick_nb(int nb) { return nb <= 1 ? 1 : (nb == 2 ? 2 : 4); }

cudaError_t launch_synthesis(const Plan& p, const double2* u, int nb, cudaStream_t s,
                             int* step_counter) {
  const int NB = pick_nb(nb);
  dim3 grid(p.T + 1, p.J / (kRowsPerWarp * p.synth_warps), (nb + NB - 1) / NB);
  dim3 block(32 * p.synth_warps);
#define SDCSW_SYN(NBV)                                                                         \
  k_synthesis<NBV><<<grid, block, 0, s>>>(u, nb, p.T, p.J, p.C, p.ptab, p.htab, p.rowoff,      \
                                          p.n_even, p.row_n, p.moff, p.inv_nn, p.radius, p.fsyn, \
                                          step_counter)
  if (NB == 1) SDCSW_SYN(1);
  else if (NB == 2) SDCSW_SYN(2);
  else SDCSW_SYN(4);
#undef SDCSW_SYN
  return cudaGetLastError();
}

cudaError_t launch_analysis(const Plan& p, double2* fe, int nb, cudaStream_t s) {
  const int NB = pick_nb(nb);
  dim3 grid(p.n_anal_work, (nb + NB - 1) / NB);
  dim3 block(32 * p.anal_warps);
#define SDCSW_ANA(NBV)                                                                         \
  k_analysis<NBV><<<grid, block, 0, s>>>(p.gan, nb, p.T, p.J, p.C, p.ptab, p.htab, p.rowoff,   \
                                         p.n_even, p.row_n, p.moff, p.lam, p.anal_work, fe)
  if (NB == 1) SDCSW_ANA(1);
  else if (NB == 2) SDCSW_ANA(2);
  else SDCSW_ANA(4);
#undef SDCSW_ANA
  return cudaGetLastError();
}

}  // namespace sdcsw
