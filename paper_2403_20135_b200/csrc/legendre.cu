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

// Both GEMMs: a CTA of kWarps warps = WJ output row tiles (16 rows each) x
// WK K-splits (WJ * WK = kWarps, chosen per plan: many K-splits for small
// truncations so enough warps are in flight, many row tiles for large ones
// so the B operand is reused through L1).  A fragments (tables) and B
// fragments (coefficients / analysis data) are loaded straight from global
// memory; the K loop has no shared-memory staging and no barriers, and is
// unrolled so its loads are issued ahead of the DMMAs.  CTAs are launched
// m-major, so all CTAs of one wavenumber run together and its B slice stays
// in L2.  Partial sums of the K-splits are reduced in shared memory in a
// fixed order (deterministic).
constexpr int kWarps = 4;

// ---------------------------------------------------------------------------
// synthesis: u [nb][3][C] -> fsyn [nb][J][L][4 (U,V,zeta,Phi)][2 (N,S)]
// grid (J / (16 WJ), T+1, ceil(nb/NB)), block 32*kWarps
// P columns: (U,V) of all b (4 NB), then (zeta,Phi) of all b; H columns: (U,V).
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(32 * kWarps) k_synthesis(
    const double2* __restrict__ u, int nb, int T, int J, int C, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, const int* __restrict__ row_n, const int* __restrict__ moff,
    const double* __restrict__ inv_nn, double radius, double2* __restrict__ fsyn,
    int* step_counter, int WJ) {
  constexpr int TH = (NB + 1) / 2;  // H tiles
  constexpr int NACC = 2 * NB * 4;  // doubles per lane (E and O, re and im)
  __shared__ double red[kWarps * 32 * NACC];

  const int m = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int WK = kWarps / WJ;
  const int jt = warp % WJ, ks = warp / WJ;
  const int j0 = (blockIdx.x * WJ + jt) * kRowsPerWarp;
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

  // this lane's B columns: P tile c holds column 8c + g
  int pb[NB], pf[NB], pr[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const int col = 8 * c + g;
    if (col < 4 * NB) { pb[c] = col >> 2; pf[c] = (col & 3) >> 1; }      // 0 = U, 1 = V
    else { pb[c] = (col - 4 * NB) >> 2; pf[c] = 2 + (((col - 4 * NB) & 3) >> 1); }  // zeta, Phi
    pr[c] = col & 1;
  }
  const double2* ub[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const int bb = b0 + pb[c] < nb ? b0 + pb[c] : -1;
    ub[c] = bb >= 0 ? u + (size_t)bb * 3 * C + mo - m : nullptr;
  }

  double accE[2][NB][2], accO[2][NB][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) accE[a][c][0] = accE[a][c][1] = accO[a][c][0] = accO[a][c][1] = 0.0;

  const int nsteps = rows >> 2;
#pragma unroll 4
  for (int s = ks; s < nsteps; s += WK) {
    const int r = 4 * s;
    const size_t off = (size_t)(r + t) * J;
    const double aP0 = __ldg(P + off), aP1 = __ldg(P + off + 8);
    const double aH0 = __ldg(H + off), aH1 = __ldg(H + off + 8);
    const int n = __ldg(row_n + r0m + r + t);
    double bP[NB], bH[TH];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      double x = 0.0, y = 0.0;
      if (n >= 0 && ub[c] != nullptr) {
        const double il = __ldg(inv_nn + mo + n - m);
        const double2* s3 = ub[c] + n;
        const int f = pf[c];
        if (f == 0) {  // U: P part i m chi / a = -i m a il delta ; H part -psi/a = a il zeta
          const double2 d = s3[2 * C];
          const double sm = dm * radius * il;
          x = pr[c] ? -sm * d.x : sm * d.y;
          if (c < TH) { const double2 z = s3[C]; y = radius * il * (pr[c] ? z.y : z.x); }
        } else if (f == 1) {  // V: P part i m psi / a ; H part chi / a = -a il delta
          const double2 z = s3[C];
          const double sm = dm * radius * il;
          x = pr[c] ? -sm * z.x : sm * z.y;
          if (c < TH) { const double2 d = s3[2 * C]; y = -radius * il * (pr[c] ? d.y : d.x); }
        } else {
          const double2 v = f == 2 ? s3[C] : s3[0];
          x = pr[c] ? v.y : v.x;
        }
      }
      bP[c] = x;
      if (c < TH) bH[c] = y;
    }
    if (r < le) {
#pragma unroll
      for (int c = 0; c < NB; ++c) { dmma(accE[0][c], aP0, bP[c]); dmma(accE[1][c], aP1, bP[c]); }
#pragma unroll
      for (int c = 0; c < TH; ++c) { dmma(accO[0][c], aH0, bH[c]); dmma(accO[1][c], aH1, bH[c]); }
    } else {
#pragma unroll
      for (int c = 0; c < NB; ++c) { dmma(accO[0][c], aP0, bP[c]); dmma(accO[1][c], aP1, bP[c]); }
#pragma unroll
      for (int c = 0; c < TH; ++c) { dmma(accE[0][c], aH0, bH[c]); dmma(accE[1][c], aH1, bH[c]); }
    }
  }
  // fixed-order reduction over the K-splits of each row tile
  if (WK > 1) {
    double* d = red + (warp * 32 + lane) * NACC;
    int q = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        d[q++] = accE[a][c][0]; d[q++] = accE[a][c][1];
        d[q++] = accO[a][c][0]; d[q++] = accO[a][c][1];
      }
    __syncthreads();
    if (ks != 0) return;
    for (int w = 1; w < WK; ++w) {
      const double* e = red + ((w * WJ + jt) * 32 + lane) * NACC;
      int qq = 0;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          accE[a][c][0] += e[qq++]; accE[a][c][1] += e[qq++];
          accO[a][c][0] += e[qq++]; accO[a][c][1] += e[qq++];
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
      f = (col & 3) >> 1;
    } else {
      b = (col - 4 * NB) >> 2;
      f = 2 + (((col - 4 * NB) & 3) >> 1);
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
// analysis: gan [nb][L][J][2 (S,A)][7] complex -> fe [nb][3][C]
// grid (n_work, ceil(nb / NB)), block 32*kWarps; work = (m << 16) | block of
// WJ 16-row tiles (m-major order)
// P columns: (phi, zeta, delta) of all b (6 NB), then ke of all b; H: first 6 NB.
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(32 * kWarps) k_analysis(
    const double2* __restrict__ gan, int nb, int T, int J, int C, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, const int* __restrict__ row_n, const int* __restrict__ moff,
    const double* __restrict__ lam, const int* __restrict__ work, double2* __restrict__ fe,
    int WJ) {
  constexpr int HU = 6 * NB;
  constexpr int TH = (HU + 7) / 8;
  constexpr int PC = 8 * NB;
  constexpr int OS = PC + 1;
  constexpr int NACC = 2 * NB * 2;
  constexpr int RED = kWarps * 32 * NACC;
  constexpr int OUT = kWarps * kRowsPerWarp * OS;
  __shared__ double red[RED > OUT ? RED : OUT];

  const int wk = work[blockIdx.x];
  const int m = wk >> 16, rb = wk & 0xffff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int WK = kWarps / WJ;
  const int rt = warp % WJ, ks = warp / WJ;
  const int b0 = blockIdx.y * NB;
  const int L = T + 1;
  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  const int rw = (rb * WJ + rt) * kRowsPerWarp;
  const bool live = rw < rows;
  const bool ev0 = rw < le, ev1 = rw + 8 < le;
  const double* P = ptab + (size_t)(r0m + rw + g) * J + t;
  const double* H = htab + (size_t)(r0m + rw + g) * J + t;

  // this lane's B columns (one per tile): data element offsets within a (b, m, j) record
  // record = [fold 0 (S): 7 complex][fold 1 (A): 7 complex] = 28 doubles
  const double* gb = reinterpret_cast<const double*>(gan);
  long long pbase[NB], hbase[TH];
  int pel[NB], hel[TH];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const int col = 8 * c + g;
    int b, slot;
    if (col < HU) { b = col / 6; slot = kXPhi + (col % 6) / 2; }
    else { b = (col - HU) >> 1; slot = kXKe; }
    pbase[c] = b0 + b < nb ? (((long long)(b0 + b) * L + m) * J) * 28 : -1;
    pel[c] = slot * 2 + (col & 1);
  }
#pragma unroll
  for (int c = 0; c < TH; ++c) {
    const int col = 8 * c + g;
    const int b = col / 6;
    hbase[c] = (col < HU && b0 + b < nb) ? (((long long)(b0 + b) * L + m) * J) * 28 : -1;
    hel[c] = (kYPhi + (col % 6) / 2) * 2 + (col & 1);
  }

  double acc[2][NB][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;

  if (live) {
    const int nsteps = J >> 2;
#pragma unroll 4
    for (int s = ks; s < nsteps; s += WK) {
      const int k = 4 * s;
      const double aP0 = __ldg(P + k), aP1 = __ldg(P + k + 8 * (size_t)J);
      const double aH0 = __ldg(H + k), aH1 = __ldg(H + k + 8 * (size_t)J);
      const long long jrec = (long long)(k + t) * 28;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        double bs = 0.0, ba = 0.0;
        if (pbase[c] >= 0) {
          bs = __ldg(gb + pbase[c] + jrec + pel[c]);
          ba = __ldg(gb + pbase[c] + jrec + 14 + pel[c]);
        }
        dmma(acc[0][c], aP0, ev0 ? bs : ba);
        dmma(acc[1][c], aP1, ev1 ? bs : ba);
      }
#pragma unroll
      for (int c = 0; c < TH; ++c) {
        double bs = 0.0, ba = 0.0;
        if (hbase[c] >= 0) {
          bs = __ldg(gb + hbase[c] + jrec + hel[c]);
          ba = __ldg(gb + hbase[c] + jrec + 14 + hel[c]);
        }
        dmma(acc[0][c], aH0, ev0 ? ba : bs);
        dmma(acc[1][c], aH1, ev1 ? ba : bs);
      }
    }
  }
  if (WK > 1) {
    double* d = red + (warp * 32 + lane) * NACC;
    int q = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < NB; ++c) { d[q++] = acc[a][c][0]; d[q++] = acc[a][c][1]; }
    __syncthreads();
    if (ks == 0) {
      for (int w = 1; w < WK; ++w) {
        const double* e = red + ((w * WJ + rt) * 32 + lane) * NACC;
        int qq = 0;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int c = 0; c < NB; ++c) { acc[a][c][0] += e[qq++]; acc[a][c][1] += e[qq++]; }
      }
    }
    __syncthreads();
  }
  if (ks != 0 || !live) return;
  double* o = red + rt * kRowsPerWarp * OS;
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

static int pick_nb(int nb) { return nb <= 6 ? nb : 4; }

#define SDCSW_NB_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6)

cudaError_t launch_synthesis(const Plan& p, const double2* u, int nb, cudaStream_t s,
                             int* step_counter) {
  const int NB = pick_nb(nb);
  const int WJ = p.synth_wj;
  dim3 grid(p.J / (kRowsPerWarp * WJ), p.T + 1, (nb + NB - 1) / NB);
#define SDCSW_SYN(NBV)                                                                           \
  if (NB == NBV) {                                                                               \
    k_synthesis<NBV><<<grid, 32 * kWarps, 0, s>>>(u, nb, p.T, p.J, p.C, p.ptab, p.htab,          \
                                                  p.rowoff, p.n_even, p.row_n, p.moff, p.inv_nn, \
                                                  p.radius, p.fsyn, step_counter, WJ);           \
    return cudaGetLastError();                                                                   \
  }
  SDCSW_NB_LIST(SDCSW_SYN)
#undef SDCSW_SYN
  return cudaErrorInvalidValue;
}

cudaError_t launch_analysis(const Plan& p, double2* fe, int nb, cudaStream_t s) {
  const int NB = pick_nb(nb);
  dim3 grid(p.n_anal_work, (nb + NB - 1) / NB);
#define SDCSW_ANA(NBV)                                                                          \
  if (NB == NBV) {                                                                              \
    k_analysis<NBV><<<grid, 32 * kWarps, 0, s>>>(p.gan, nb, p.T, p.J, p.C, p.ptab, p.htab,      \
                                                 p.rowoff, p.n_even, p.row_n, p.moff, p.lam,    \
                                                 p.anal_work, fe, p.anal_wj);                   \
    return cudaGetLastError();                                                                  \
  }
  SDCSW_NB_LIST(SDCSW_ANA)
#undef SDCSW_ANA
  return cudaErrorInvalidValue;
}

}  // namespace sdcsw
