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
#include "node_math.cuh"

#ifndef SDCSW_EPI_PRELOAD
#define SDCSW_EPI_PRELOAD 1  // fused epilogue node data loaded before the split-K reduction
#endif
#ifndef SDCSW_EXP
#define SDCSW_EXP 0
#endif
#ifndef SDCSW_SYN_MB1
#define SDCSW_SYN_MB1 5  // synthesis NB <= 2: 5 CTAs per SM (one wave at T127; measured)
#endif
#if SDCSW_EXP == 5
__device__ long long g_ph[8 * 4096];
extern "C" int sdcsw_debug_phases(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_ph, n * sizeof(long long));
}
#define PH(i) if (threadIdx.x == 0 && blockIdx.x < 4096 && blockIdx.y == 0) { g_ph[8 * blockIdx.x + (i)] = clock64(); \
  if ((i) == 0 || (i) == 4) { unsigned long long gt; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt)); \
    g_ph[8 * blockIdx.x + 5 + ((i) == 4)] = (long long)gt; } \
  if ((i) == 0) { unsigned sm; asm volatile("mov.u32 %0, %smid;" : "=r"(sm)); g_ph[8 * blockIdx.x + 7] = sm; } }
#else
#define PH(i)
#endif
#if SDCSW_EXP == 3
__device__ unsigned long long g_times[1 << 17];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
extern "C" int sdcsw_debug_times(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_times, n * sizeof(unsigned long long));
}
#endif

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
// synthesis B-operand prep for API calls: xsyn record per (valid row, b)
// grid (ceil(2C/256), nb): one thread per (coefficient, re/im, batch entry)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_synth_prep(const double* __restrict__ u, int C2, int nb,
                                                    const double2* __restrict__ xscale,
                                                    const int* __restrict__ idx_row,
                                                    double* __restrict__ xsyn, int rows, int chunk,
                                                    const int* __restrict__ idx_list, int n_list) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx_list != nullptr) {  // spectral split: own coefficients only
    if (e >= 2 * n_list) return;
    e = 2 * idx_list[e >> 1] + (e & 1);
  }
  if (e >= C2) return;
  const int b = blockIdx.y;
  const double* s = u + (size_t)b * 3 * C2;
  const int idx = e >> 1;
  const int ch = chunk > 0 ? chunk : nb;  // chunk-major record layout (see f_expl_prepped)
  const int cb = b / ch, w = nb - cb * ch < ch ? nb - cb * ch : ch;
  double* rec = xsyn + (size_t)cb * rows * ch * kXsyn + xsyn_off(idx_row[idx], b - cb * ch, w);
  write_xsyn_half(rec, 16 * (size_t)w, e & 1, s[e], s[C2 + e], s[2 * C2 + e], xscale[idx]);
}

// ---------------------------------------------------------------------------
// synthesis: xsyn -> fsyn [nb][J][L][4 (U,V,zeta,Phi)][2 (N,S)]
// grid (J / (16 WJ), T+1, ceil(nb / (NB NBC))), block 32 WJ WK
// Batch entries are taken in pairs (b, b+1).  Column tile 2p of pair p holds
// (U, V) x (re, im) of both entries, tile 2p + 1 their (zeta, Phi); the H-table
// contribution (U and V only) has exactly the (U, V) tile's columns, so it
// accumulates into the same registers - no zero columns, no extra accumulators.
// A CTA loops over NBC batch blocks of NB entries; its table slice is then
// re-read from L1 instead of being re-fetched by a separate CTA per block.
// ---------------------------------------------------------------------------
template <int NB, int PF>
#ifndef SDCSW_SYN_MINB
#define SDCSW_SYN_MINB 4
#endif
// NB <= 4: cap the registers at 128 so that 4 CTAs fit per SM - the c1 sweep
// analysis (576 CTAs) then runs in one wave (measured)
#define SDCSW_ANA_LB __launch_bounds__(32 * kWarps) __maxnreg__(NB == 1 && !FZ ? 64 : (NB <= 4 ? 128 : 255))
__global__ void __launch_bounds__(32 * kWarps, NB <= 2 ? SDCSW_SYN_MB1 : (NB <= 4 ? SDCSW_SYN_MINB : 3)) k_synthesis(
    const double* __restrict__ xsyn, int nb, int T, int J, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, double2* __restrict__ fsyn, int* step_counter, int WJ,
    int NBC, const int* __restrict__ mlist, int Lp, const SynDst sd) {
  SDCSW_PDL_ENTRY();
  if (SDCSW_TRIG_SYN == 1) SDCSW_PDL_TRIGGER();
  constexpr int NPAIR = (NB + 1) / 2;
  constexpr int NT = 2 * NPAIR;     // column tiles: (U,V) and (zeta,Phi) per pair
  constexpr int NACC = NT * 2 * 4;  // doubles per lane: tiles x row tiles x (E,O) x (re,im)
  __shared__ double red[2 * 32 * NACC];  // two warps' partials (tree reduction)

  // unsplit: m = k = blockIdx.y, Lp = T + 1; spectral split: m = own list[k]
  const int kpos = blockIdx.y;
  const int m = mlist != nullptr ? mlist[kpos] : kpos;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int WK = (blockDim.x >> 5) / WJ;
  const int jt = warp % WJ, ks = warp / WJ;
  const int j0 = (blockIdx.x * WJ + jt) * kRowsPerWarp;
  (void)T;
  // constant plan data before the dependency wait (overlaps the producer's tail)
  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  SDCSW_PDL_WAIT();
  if (step_counter != nullptr && (blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) == 0)
    atomicAdd(step_counter, 1);
  // fragment-order tables ([rows/4][J/8][8][4], lane order): lane (g, t) of
  // k-step s reads row r0m + 4 s + t, latitudes j0 + g and j0 + 8 + g; a warp
  // load is 256 contiguous bytes
  const size_t qstride = (size_t)(J / 8) * 32;
  const double* P = ptab + ((size_t)(r0m / 4) * (J / 8) + j0 / 8) * 32 + g * 4 + t;
  const double* H = htab + ((size_t)(r0m / 4) * (J / 8) + j0 / 8) * 32 + g * 4 + t;
  const size_t qstep = (size_t)3 * nb * 16;  // one row quad (k-step) of the operand
  const size_t pstr = (size_t)16 * nb;         // part stride
  const int nsteps = rows >> 2;
  const int se = le >> 2;  // steps [0, se) are even-class rows
  const int gb = g >> 2, gc = g & 3;  // lane's entry within the pair, column within the entry

  for (int bb = 0; bb < NBC; ++bb) {
    const int b0 = (blockIdx.z * NBC + bb) * NB;
    if (b0 >= nb) break;
    const int nbv = nb - b0 < NB ? nb - b0 : NB;
    // fragment-order operand: lane (g, t) of k-step s reads row quad r0m/4 + s,
    // row t, entry b0 + 2p + gb, column gc - 32 consecutive doubles per warp load
    const double* X = xsyn + (size_t)(r0m / 4) * qstep + (size_t)b0 * 16 + t * 4 + gc;

    double aE[2][NT][2], aO[2][NT][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < NT; ++c) aE[a][c][0] = aE[a][c][1] = aO[a][c][0] = aO[a][c][1] = 0.0;

    // K loop in two branch-free ranges (even rows, then odd rows); fragments of
    // step s + PF WK are loaded before the DMMAs of step s
    struct Frag {
      double aP0, aP1, aH0, aH1, bP[NT], bH[NPAIR];
    };
    auto fetch = [&](int s, Frag& f) {
      const size_t off = (size_t)s * qstride;
      f.aP0 = __ldg(P + off);
      f.aP1 = __ldg(P + off + 32);
      f.aH0 = __ldg(H + off);
      f.aH1 = __ldg(H + off + 32);
      const double* rec = X + (size_t)s * qstep;
#pragma unroll
      for (int p = 0; p < NPAIR; ++p) {
        const int be = 2 * p + gb;
        const bool ok = be < nbv;
        const double* rb = rec + be * 16;
        f.bP[2 * p] = ok ? __ldg(rb) : 0.0;                // U, V (P part)
        f.bP[2 * p + 1] = ok ? __ldg(rb + pstr) : 0.0;     // zeta, Phi
        f.bH[p] = ok ? __ldg(rb + 2 * pstr) : 0.0;         // U, V (H part)
      }
    };
#pragma unroll
    for (int cls = 0; cls < 2; ++cls) {
      const int lo = cls == 0 ? 0 : se, hi = cls == 0 ? se : nsteps;
      int s = lo + ((ks - lo) % WK + WK) % WK;  // first step of this warp in [lo, hi)
      if (s >= hi) continue;
      Frag cur, nx1, nx2;
      fetch(s, cur);
      if (PF == 2) fetch(s + WK < hi ? s + WK : s, nx1);
      for (; s < hi; s += WK) {
        const int sn = s + PF * WK < hi ? s + PF * WK : s;  // clamped: always a valid address
        fetch(sn, PF == 2 ? nx2 : nx1);
        if (cls == 0) {  // n - m even: P symmetric (E), H antisymmetric (O)
#pragma unroll
          for (int c = 0; c < NT; ++c) { dmma(aE[0][c], cur.aP0, cur.bP[c]); dmma(aE[1][c], cur.aP1, cur.bP[c]); }
#pragma unroll
          for (int p = 0; p < NPAIR; ++p) { dmma(aO[0][2 * p], cur.aH0, cur.bH[p]); dmma(aO[1][2 * p], cur.aH1, cur.bH[p]); }
        } else {
#pragma unroll
          for (int c = 0; c < NT; ++c) { dmma(aO[0][c], cur.aP0, cur.bP[c]); dmma(aO[1][c], cur.aP1, cur.bP[c]); }
#pragma unroll
          for (int p = 0; p < NPAIR; ++p) { dmma(aE[0][2 * p], cur.aH0, cur.bH[p]); dmma(aE[1][2 * p], cur.aH1, cur.bH[p]); }
        }
        cur = nx1;
        if (PF == 2) nx1 = nx2;
      }
    }
    if (SDCSW_TRIG_SYN == 2) SDCSW_PDL_TRIGGER();
    // fixed-order tree reduction over the K-splits ((w0 + w2) + (w1 + w3));
    // lane-fastest layout, conflict-free
    bool owner = true;
    if (WK > 1) {
      for (int half = WK / 2; half >= 1; half /= 2) {
        __syncthreads();  // `red` is free
        if (ks >= half && ks < 2 * half) {
          double* d = red + ((ks - half) * WJ + jt) * NACC * 32 + lane;
          int q = 0;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int c = 0; c < NT; ++c) {
              d[32 * q++] = aE[a][c][0]; d[32 * q++] = aE[a][c][1];
              d[32 * q++] = aO[a][c][0]; d[32 * q++] = aO[a][c][1];
            }
        }
        __syncthreads();
        if (ks < half) {
          const double* e = red + (ks * WJ + jt) * NACC * 32 + lane;
          int q = 0;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int c = 0; c < NT; ++c) {
              aE[a][c][0] += e[32 * q++]; aE[a][c][1] += e[32 * q++];
              aO[a][c][0] += e[32 * q++]; aO[a][c][1] += e[32 * q++];
            }
        }
      }
      owner = ks == 0;
    }
    if (owner && j0 < J) {
      // epilogue: lane (g, t) of tile c holds batch b0 + 2 (c/2) + (t >> 1),
      // field (t & 1) + 2 (c & 1)  (U, V, zeta, Phi)
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        const int be = 2 * (c >> 1) + (t >> 1);
        const int f = (t & 1) + 2 * (c & 1);
        if (be >= nbv) continue;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int j = j0 + 8 * a + g;
          const size_t off = ((((size_t)(b0 + be) * J + j) * Lp + kpos) * 4 + f) * 2;
          const double2 vn = make_double2(aE[a][c][0] + aO[a][c][0], aE[a][c][1] + aO[a][c][1]);
          const double2 vs = make_double2(aE[a][c][0] - aO[a][c][0], aE[a][c][1] - aO[a][c][1]);
          if (sd.n == 0) {
            fsyn[off] = vn;
            fsyn[off + 1] = vs;
          } else {  // spectral split over peer memory: every spectral peer's buffer
            const long long par = (long long)((*sd.fseq + 1) & 1) * sd.par_stride;
            for (int q = 0; q < sd.n; ++q) {
              sd.dst[q][par + off] = vn;
              sd.dst[q][par + off + 1] = vs;
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Synthesis with a per-warp cp.async pipeline: the A (table) and B (operand)
// fragments of a warp's next kSynStages-1 k-steps are in flight as async copies
// into shared memory (no registers held), so the K loop is no longer bound by
// one L2 round trip per k-step.  Same arithmetic and reduction as k_synthesis.
// ---------------------------------------------------------------------------
#ifndef SDCSW_SYN_STAGES
#define SDCSW_SYN_STAGES 3
#endif
constexpr int kSynStages = SDCSW_SYN_STAGES;
template <int NB>
constexpr int syn_stage_doubles() { return 128 + 96 * ((NB + 1) / 2); }
template <int NB>
constexpr size_t syn_cp_smem() { return (size_t)kWarps * kSynStages * syn_stage_doubles<NB>() * 8; }

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool valid = true) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NB>
__global__ void __launch_bounds__(32 * kWarps, NB <= 2 ? SDCSW_SYN_MB1 : (NB <= 4 ? SDCSW_SYN_MINB : 3)) k_synthesis_cp(
    const double* __restrict__ xsyn, int nb, int T, int J, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, double2* __restrict__ fsyn, int* step_counter, int WJ,
    int NBC, const int* __restrict__ mlist, int Lp, const SynDst sd) {
  SDCSW_PDL_ENTRY();
  constexpr int NPAIR = (NB + 1) / 2;
  constexpr int NT = 2 * NPAIR;
  constexpr int NACC = NT * 2 * 4;
  constexpr int STG = syn_stage_doubles<NB>();
  __shared__ double red[2 * 32 * NACC];
  extern __shared__ __align__(16) double synstage[];  // [warp][kSynStages][STG]

  const int kpos = blockIdx.y;
  const int m = mlist != nullptr ? mlist[kpos] : kpos;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int WK = (blockDim.x >> 5) / WJ;
  const int jt = warp % WJ, ks = warp / WJ;
  const int j0 = (blockIdx.x * WJ + jt) * kRowsPerWarp;
  (void)T;
  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  SDCSW_PDL_WAIT();
  if (step_counter != nullptr && (blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) == 0)
    atomicAdd(step_counter, 1);
  const size_t qstride = (size_t)(J / 8) * 32;
  const double* Pb = ptab + ((size_t)(r0m / 4) * (J / 8) + j0 / 8) * 32;
  const double* Hb = htab + ((size_t)(r0m / 4) * (J / 8) + j0 / 8) * 32;
  const size_t qstep = (size_t)3 * nb * 16;
  const size_t pstr = (size_t)16 * nb;
  const int nsteps = rows >> 2;
  const int se = le >> 2;
  const int gb = g >> 2, gc = g & 3;
  double* mys = synstage + warp * kSynStages * STG;
  const int nk = ks < nsteps ? (nsteps - ks + WK - 1) / WK : 0;  // this warp's k-steps

  for (int bb = 0; bb < NBC; ++bb) {
    const int b0 = (blockIdx.z * NBC + bb) * NB;
    if (b0 >= nb) break;
    const int nbv = nb - b0 < NB ? nb - b0 : NB;
    const double* Xb = xsyn + (size_t)(r0m / 4) * qstep + (size_t)b0 * 16;
    double aE[2][NT][2], aO[2][NT][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < NT; ++c) aE[a][c][0] = aE[a][c][1] = aO[a][c][0] = aO[a][c][1] = 0.0;

    // stage of this warp's k-th step: [P: 64][H: 64][operand: 3 parts x NPAIR pairs x 32]
    auto issue = [&](int k) {
      if (k < nk) {
        const int s = ks + k * WK;
        double* st = mys + (k % kSynStages) * STG;
        cp_async16(st + 2 * lane, Pb + s * qstride + 2 * lane);
        cp_async16(st + 64 + 2 * lane, Hb + s * qstride + 2 * lane);
        const double* xq = Xb + (size_t)s * qstep;
        for (int ci = lane; ci < 3 * NPAIR * 16; ci += 32) {
          const int q = ci / (NPAIR * 16), r2 = ci - q * NPAIR * 16, p = r2 >> 4, w = r2 & 15;
          cp_async16(st + 128 + (q * NPAIR + p) * 32 + 2 * w, xq + q * pstr + p * 32 + 2 * w,
                     2 * p + (w >> 3) < nbv);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < kSynStages - 1; ++k) issue(k);
    for (int k = 0; k < nk; ++k) {
      issue(k + kSynStages - 1);
      cp_async_wait<kSynStages - 1>();
      __syncwarp();
      const double* st = mys + (k % kSynStages) * STG;
      const double aP0 = st[lane], aP1 = st[32 + lane], aH0 = st[64 + lane], aH1 = st[96 + lane];
      double bP[NT], bH[NPAIR];
#pragma unroll
      for (int p = 0; p < NPAIR; ++p) {
        const double* bq = st + 128 + p * 32 + gb * 16 + t * 4 + gc;
        bP[2 * p] = bq[0];
        bP[2 * p + 1] = bq[NPAIR * 32];
        bH[p] = bq[2 * NPAIR * 32];
      }
      if (ks + k * WK < se) {  // n - m even: P symmetric (E), H antisymmetric (O)
#pragma unroll
        for (int c = 0; c < NT; ++c) { dmma(aE[0][c], aP0, bP[c]); dmma(aE[1][c], aP1, bP[c]); }
#pragma unroll
        for (int p = 0; p < NPAIR; ++p) { dmma(aO[0][2 * p], aH0, bH[p]); dmma(aO[1][2 * p], aH1, bH[p]); }
      } else {
#pragma unroll
        for (int c = 0; c < NT; ++c) { dmma(aO[0][c], aP0, bP[c]); dmma(aO[1][c], aP1, bP[c]); }
#pragma unroll
        for (int p = 0; p < NPAIR; ++p) { dmma(aE[0][2 * p], aH0, bH[p]); dmma(aE[1][2 * p], aH1, bH[p]); }
      }
      __syncwarp();  // the stage is refilled by a later issue()
    }
    cp_async_wait<0>();
    bool owner = true;
    if (WK > 1) {
      for (int half = WK / 2; half >= 1; half /= 2) {
        __syncthreads();
        if (ks >= half && ks < 2 * half) {
          double* d = red + ((ks - half) * WJ + jt) * NACC * 32 + lane;
          int q = 0;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int c = 0; c < NT; ++c) {
              d[32 * q++] = aE[a][c][0]; d[32 * q++] = aE[a][c][1];
              d[32 * q++] = aO[a][c][0]; d[32 * q++] = aO[a][c][1];
            }
        }
        __syncthreads();
        if (ks < half) {
          const double* e = red + (ks * WJ + jt) * NACC * 32 + lane;
          int q = 0;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int c = 0; c < NT; ++c) {
              aE[a][c][0] += e[32 * q++]; aE[a][c][1] += e[32 * q++];
              aO[a][c][0] += e[32 * q++]; aO[a][c][1] += e[32 * q++];
            }
        }
      }
      owner = ks == 0;
    }
    if (owner && j0 < J) {
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        const int be = 2 * (c >> 1) + (t >> 1);
        const int f = (t & 1) + 2 * (c & 1);
        if (be >= nbv) continue;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int j = j0 + 8 * a + g;
          const size_t off = ((((size_t)(b0 + be) * J + j) * Lp + kpos) * 4 + f) * 2;
          const double2 vn = make_double2(aE[a][c][0] + aO[a][c][0], aE[a][c][1] + aO[a][c][1]);
          const double2 vs = make_double2(aE[a][c][0] - aO[a][c][0], aE[a][c][1] - aO[a][c][1]);
          if (sd.n == 0) {
            fsyn[off] = vn;
            fsyn[off + 1] = vs;
          } else {  // spectral split over peer memory: every spectral peer's buffer
            const long long par = (long long)((*sd.fseq + 1) & 1) * sd.par_stride;
            for (int q = 0; q < sd.n; ++q) {
              sd.dst[q][par + off] = vn;
              sd.dst[q][par + off + 1] = vs;
            }
          }
        }
      }
    }
  }
}

#define SDCSW_NB_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6)
cudaError_t configure_synthesis() {
  cudaError_t e = cudaSuccess;
#define SDCSW_SYN_CFG(NBV)                                                                        \
  if (e == cudaSuccess)                                                                          \
    e = cudaFuncSetAttribute(k_synthesis_cp<NBV>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                             (int)syn_cp_smem<NBV>());
  SDCSW_NB_LIST(SDCSW_SYN_CFG)
#undef SDCSW_SYN_CFG
  return e;
}

// ---------------------------------------------------------------------------
// analysis: gan [nb][L][J][2 (S,A)][7] complex -> fe [nb][3][C]
// grid (n_work, ceil(nb / NB)), block 32*kWarps; work = (m << 16) | block of
// WJ 16-row tiles (m-major order)
// P columns: (phi, zeta, delta) of all b (6 NB), then ke of all b; H: first 6 NB.
// ---------------------------------------------------------------------------
// Sweep-fused epilogue (FuseArgs, internal.cuh).  Lane (rr, ri) of the warp's
// 16-row output tile owns one real component of one coefficient for all M
// nodes: it forms f_E of each node from the tile (the plain epilogue's
// arithmetic), then the node update of k_sweep_nodes / k_final_node (nodes.cu)
// in the same rounded order, so results are bit-identical to the unfused step.
template <int NB>
__device__ __forceinline__ void fused_nodes(const FuseArgs& fz, const double* o, int n, int mo,
                                            int m, int C, const double* __restrict__ lamv,
                                            const double2* __restrict__ xscale, double* stage,
                                            int lane, int b0, int nb, const Tri& pre_a0,
                                            const Tri* pre_fi, double pre_l, double2 pre_sc) {
  constexpr int OS = 8 * NB + 1;
  constexpr int MX = kFuseMaxNodes;
  const int rr = lane & 15, ri = lane >> 4;
  if (n < 0) return;
  const int idx = mo + n - m;
  const int C2 = 2 * C, e = 2 * idx + ri;
  const size_t S2 = 3 * (size_t)C2;
  const double* row = o + rr * OS;
  const bool pre = SDCSW_EPI_PRELOAD && (fz.mode == 1 || fz.mode == 2);
  const double l = pre ? pre_l : lamv[idx];
  const bool zero = m == 0 && ri == 1;
  Tri fe[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    fe[b].phi = zero ? 0.0 : row[6 * b + ri];
    fe[b].zeta = zero ? 0.0 : row[6 * b + 2 + ri];
    fe[b].delta = zero ? 0.0 : __fma_rn(l, row[6 * NB + 2 * b + ri], row[6 * b + 4 + ri]);
  }
  if (fz.mode == 4) {  // node-parallel: publish (fe, fi) of this rank's nodes to every rank
    const long long par = (long long)(exchange_number(fz.peer_epoch, fz.peer_k, fz.peer_kx) & 1);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (b0 + b >= nb) break;
      const Tri fi = load_tri(fz.peer_fi + (size_t)(b0 + b) * S2, C2, e);
      const size_t slot = ((size_t)par * fz.M + fz.peer_lo + b0 + b) * 2 * S2;
      for (int q = 0; q < fz.peer_world; ++q) {
        store_tri(fz.peer_x[q] + slot, C2, e, fe[b]);
        store_tri(fz.peer_x[q] + slot + S2, C2, e, fi);
      }
    }
    return;  // posted by the consumer after this grid completed (peer_wait)
  }
  if (fz.mode == 3) {  // serial SDC: store fe_m, serial_update(m), serial_node(m + 1)
    store_tri(fz.fe_new, C2, e, fe[0]);
    if (fz.quad_next == nullptr) return;
    const Tri a0 = load_tri(fz.u0, C2, e);
    const Tri fi0 = f_impl_tri(a0, fz.phibar, l);
    const Tri eo = load_tri(fz.fe_old, C2, e);
    const Tri fn = load_tri(fz.fi_new, C2, e);
    const Tri fo = fz.first ? fi0 : load_tri(fz.fi_old, C2, e);
    const Tri de = sub_tri(fe[0], eo), di = sub_tri(fn, fo);
    const double we = fz.cf[0], wi = fz.cf[1];
    Tri c;
    if (fz.use_corr) {
      c = axpy_tri(load_tri(fz.corr, C2, e), we, de);
    } else {
      c = Tri{__dmul_rn(we, de.phi), __dmul_rn(we, de.zeta), __dmul_rn(we, de.delta)};
    }
    const Tri corr = axpy_tri(c, wi, di);
    store_tri(fz.corr, C2, e, corr);
    // node m + 1: beta = quad + corr - alpha fi_old; u = solve; fi_new = f_I(u)
    Tri b = add_tri(load_tri(fz.quad_next, C2, e), corr);
    const Tri fo2 = fz.first ? fi0 : load_tri(fz.fi_old_next, C2, e);
    b = axmy_tri(b, fz.cf[2], fo2);
    const Tri u = solve_tri(b, fz.cf[2], fz.cf[3], fz.cf[4], l);
    store_tri(fz.fi_new_next, C2, e, f_impl_tri(u, fz.phibar, l));
    if (fz.u_out != nullptr) {
      store_tri(fz.u_out, C2, e, u);
      if (fz.diverged != nullptr && !finite_tri(u))
        atomicMin(fz.diverged, fz.step_counter ? *fz.step_counter : 1);
    }
    write_xsyn_half(stage + xsyn_off(rr, 0, 1), 16, ri, u.phi, u.zeta, u.delta, xscale[idx]);
    return;
  }
  const int M = fz.M;
  const Tri a0 = SDCSW_EPI_PRELOAD ? pre_a0 : load_tri(fz.u0, C2, e);
  const Tri fi0 = f_impl_tri(a0, fz.phibar, l);
  Tri fi[MX];
#pragma unroll
  for (int j = 0; j < MX; ++j)
    if (j < M) fi[j] = fz.first ? fi0 : (SDCSW_EPI_PRELOAD ? pre_fi[j] : load_tri(fz.fi + j * S2, C2, e));
  if (fz.mode == 1) {
    const double2 sc = pre ? pre_sc : xscale[idx];
#pragma unroll
    for (int q = 0; q < MX; ++q) {
      if (q >= M) break;
      const double* c = fz.cf + q * (M + 4);
      Tri b = a0;
#pragma unroll
      for (int j = 0; j < MX; ++j)
        if (j < M) b = axpy_tri(b, c[j], add_tri(fe[j < NB ? j : NB - 1], fi[j]));
      b = axmy_tri(b, c[M], fi[q]);
      const Tri u = solve_tri(b, c[M + 1], c[M + 2], c[M + 3], l);
      store_tri(fz.fi + q * S2, C2, e, f_impl_tri(u, fz.phibar, l));
      write_xsyn_half(stage + xsyn_off(rr, q, M), 16 * (size_t)M, ri, u.phi, u.zeta, u.delta, sc);
    }
  } else {
    const double* c = fz.cf;
    Tri b = a0, fil = fi0;
#pragma unroll
    for (int j = 0; j < MX; ++j)
      if (j < M) {
        b = axpy_tri(axpy_tri(b, c[j], fe[j < NB ? j : NB - 1]), c[j], fi[j]);
        fil = fi[j];
      }
    b = axmy_tri(b, c[M], fil);
    const Tri u = solve_tri(b, c[M + 1], c[M + 2], c[M + 3], l);
    store_tri(fz.u_out, C2, e, u);
    if (fz.diverged != nullptr && !finite_tri(u))
      atomicMin(fz.diverged, fz.step_counter ? *fz.step_counter : 1);
    write_xsyn_half(stage + xsyn_off(rr, 0, 1), 16, ri, u.phi, u.zeta, u.delta,
                    pre ? pre_sc : xscale[idx]);
  }
}

template <int NB, int PF, bool FZ>
__global__ void SDCSW_ANA_LB k_analysis(
    const double2* __restrict__ gan, int nb, int T, int J, int C, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, const int* __restrict__ row_n, const int* __restrict__ moff,
    const double* __restrict__ lam, const int* __restrict__ work, double2* __restrict__ fe,
    int WJ, const FuseArgs fz, const double2* __restrict__ xscale, const int* __restrict__ idx_row) {
  SDCSW_PDL_ENTRY();
  PH(0)
  if (SDCSW_TRIG_ANA == 1) SDCSW_PDL_TRIGGER();
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
  // fragment-order tables ([rows/8][J/4][8][4]): lane (g, t) of k-step s reads
  // rows r0m + rw + g (+ 8), latitude 4 s + t; a warp load is 256 bytes
  const size_t tstride = (size_t)(J / 4) * 32;
  const double* P = ptab + (size_t)((r0m + rw) / 8) * tstride + g * 4 + t;
  const double* H = htab + (size_t)((r0m + rw) / 8) * tstride + g * 4 + t;

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

  // fused epilogue: this lane's degree n (constant plan data, read ahead of the GEMM)
  int fn = -1, fmo = 0;
  if constexpr (FZ) {
    const int rr = lane & 15;
    if (live && ks == 0 && rw + rr < rows) {
      fn = row_n[r0m + rw + rr];
      fmo = moff[m];
    }
  }

  if (live) {
    // fragments of step s + WK are loaded before the DMMAs of step s
    struct Frag {
      double aP0, aP1, aH0, aH1, bPs[NB], bPa[NB], bHs[TH], bHa[TH];
    };
    auto fetchA = [&](int s, Frag& f) {
      const size_t k = (size_t)s * 32;
      f.aP0 = __ldg(P + k);
      f.aP1 = __ldg(P + k + tstride);
      f.aH0 = __ldg(H + k);
      f.aH1 = __ldg(H + k + tstride);
    };
    // only the folds this warp's parity classes use are read (warp-uniform): a
    // single-class tile (the common case) reads half of each record
    const bool any_ev = ev0 || ev1, any_od = !ev0 || !ev1;
    auto fetchB = [&](int s, Frag& f) {
      const int k = 4 * s;
      const long long jrec = (long long)(k + t) * 28;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const bool ok = pbase[c] >= 0;
        f.bPs[c] = ok && any_ev ? __ldg(gb + pbase[c] + jrec + pel[c]) : 0.0;
        f.bPa[c] = ok && any_od ? __ldg(gb + pbase[c] + jrec + 14 + pel[c]) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < TH; ++c) {
        const bool ok = hbase[c] >= 0;
        f.bHs[c] = ok && any_od ? __ldg(gb + hbase[c] + jrec + hel[c]) : 0.0;
        f.bHa[c] = ok && any_ev ? __ldg(gb + hbase[c] + jrec + 14 + hel[c]) : 0.0;
      }
    };
    auto fetch = [&](int s, Frag& f) { fetchA(s, f); fetchB(s, f); };
    const int nsteps = J >> 2;
    int s = ks;
    Frag cur, nx1, nx2;
    // table fragments and plan data are constant: loaded before the dependency wait
    if (s < nsteps) fetchA(s, cur);
    SDCSW_PDL_WAIT();
    PH(1)
    if (s < nsteps) {
      fetchB(s, cur);
      if (PF == 2) fetch(s + WK < nsteps ? s + WK : s, nx1);
      for (; s < nsteps; s += WK) {
        fetch(s + PF * WK < nsteps ? s + PF * WK : s, PF == 2 ? nx2 : nx1);
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          dmma(acc[0][c], cur.aP0, ev0 ? cur.bPs[c] : cur.bPa[c]);
          dmma(acc[1][c], cur.aP1, ev1 ? cur.bPs[c] : cur.bPa[c]);
        }
#pragma unroll
        for (int c = 0; c < TH; ++c) {
          dmma(acc[0][c], cur.aH0, ev0 ? cur.bHa[c] : cur.bHs[c]);
          dmma(acc[1][c], cur.aH1, ev1 ? cur.bHa[c] : cur.bHs[c]);
        }
        cur = nx1;
        if (PF == 2) nx1 = nx2;
      }
    }
  }
  if (SDCSW_TRIG_ANA == 2) SDCSW_PDL_TRIGGER();
  // fused epilogue (modes 1, 2): the node data (u0, f_I of every node) are
  // loaded now, so their latency overlaps the split-K reduction
  Tri pre_a0{}, pre_fi[FZ ? kFuseMaxNodes : 1];
  double pre_l = 0.0;
  double2 pre_sc = make_double2(0.0, 0.0);
  if constexpr (FZ) {
    if (SDCSW_EPI_PRELOAD && fn >= 0 && (fz.mode == 1 || fz.mode == 2)) {
      const int C2 = 2 * C;
      const int idx = fmo + fn - m;
      const int e = 2 * idx + (lane >> 4);
      pre_l = lam[idx];
      pre_sc = xscale[idx];
      pre_a0 = load_tri(fz.u0, C2, e);
      if (!fz.first) {
#pragma unroll
        for (int j = 0; j < kFuseMaxNodes; ++j)
          if (j < fz.M) pre_fi[j] = load_tri(fz.fi + (size_t)j * 3 * C2, C2, e);
      }
    }
  }
  PH(2)
  if (WK > 1) {  // lane-fastest layout: conflict-free shared-memory traffic
    double* d = red + warp * NACC * 32 + lane;
    int q = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < NB; ++c) { d[32 * q++] = acc[a][c][0]; d[32 * q++] = acc[a][c][1]; }
    __syncthreads();
    if (ks == 0) {
      for (int w = 1; w < WK; ++w) {
        const double* e = red + (w * WJ + rt) * NACC * 32 + lane;
        int qq = 0;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int c = 0; c < NB; ++c) { acc[a][c][0] += e[32 * qq++]; acc[a][c][1] += e[32 * qq++]; }
      }
    }
    __syncthreads();
  }
  PH(3)
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
  if constexpr (FZ) {
    // next synthesis operand: the tile's rows r0m + rw .. are consecutive operand
    // records, staged in shared memory (zero for padding rows) and written out
    // with coalesced 16-byte stores
    __shared__ alignas(16) double xstage[2][kRowsPerWarp * kFuseMaxNodes * kXsyn];
    double* stage = xstage[rt & 1];
    const int per = (fz.mode == 1 ? fz.M : 1) * kXsyn;  // doubles per tile row
    const bool writes_operand = fz.mode != 4 && (fz.mode != 3 || fz.quad_next != nullptr);
    if (writes_operand)
      for (int i = lane; i < kRowsPerWarp * per; i += 32) stage[i] = 0.0;
    __syncwarp();
    fused_nodes<NB>(fz, o, fn, fmo, m, C, lam, xscale, stage, lane, b0, nb, pre_a0, pre_fi,
                    pre_l, pre_sc);
    __syncwarp();
    const int nrow = rows - rw < kRowsPerWarp ? rows - rw : kRowsPerWarp;
    double2* dst = reinterpret_cast<double2*>(fz.xsyn + (size_t)(r0m + rw) * per);
    const double2* src = reinterpret_cast<const double2*>(stage);
    if (writes_operand)
      for (int i = lane; i < nrow * per / 2; i += 32) dst[i] = src[i];
    PH(4)
  } else {
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
    double2 delta = make_double2(__fma_rn(l, row[6 * NB + 2 * b], row[6 * b + 4]),
                                 __fma_rn(l, row[6 * NB + 2 * b + 1], row[6 * b + 5]));
    if (m == 0) phi.y = zeta.y = delta.y = 0.0;
    double2* dst = fe + (size_t)(b0 + b) * 3 * C;
    dst[idx] = phi;
    dst[C + idx] = zeta;
    dst[2 * C + idx] = delta;
  }
  }
}

static int pick_nb(int nb) { return nb <= 6 ? nb : 4; }


cudaError_t launch_synth_prep(const Plan& p, const double2* u, int nb, double* xsyn,
                              cudaStream_t s, int chunk) {
  const int n = p.own_idx ? p.n_own_idx : p.C;
  launch_k(k_synth_prep, dim3((2 * n + 255) / 256, nb), 256, 0, s, 
      reinterpret_cast<const double*>(u), 2 * p.C, nb, p.xscale, p.idx_row, xsyn, p.rows, chunk, p.own_idx,
           p.n_own_idx);
  return cudaGetLastError();
}

static cudaError_t synthesis_impl(const Plan& p, double2* fsyn, const int* mlist, int nm, int Lp,
                                  const double* xsyn, int nb, cudaStream_t s, int* step_counter,
                                  const SynDst& sd);

// (H-free plans, ponly_on: operand conversion + P-only synthesis, legendre_ponly.cu)
cudaError_t launch_synthesis(const Plan& p, const Work& w, const double* xsyn, int nb,
                             cudaStream_t s, int* step_counter) {
  if (ponly_on(p))
    return launch_synthesis_ponly(p, w.fsyn, nullptr, p.T + 1, p.T + 1, w.xsp, xsyn, nb, s,
                                  step_counter, SynDst{});
  return synthesis_impl(p, w.fsyn, nullptr, p.T + 1, p.T + 1, xsyn, nb, s, step_counter, SynDst{});
}

cudaError_t launch_synthesis_split(const Plan& p, const double* xsyn, int nb, cudaStream_t s) {
  double2* part = p.fsyn_ext + (size_t)p.split_sp * nb * p.J * p.Lp * 8;
  if (ponly_on(p))
    return launch_synthesis_ponly(p, part, p.own_m, p.n_own_m, p.Lp, p.xsynP, xsyn, nb, s, nullptr,
                                  SynDst{});
  return synthesis_impl(p, part, p.own_m, p.n_own_m, p.Lp, xsyn, nb, s, nullptr, SynDst{});
}

cudaError_t launch_synthesis_peer(const Plan& p, const double* xsyn, int nb, cudaStream_t s,
                                  const SynDst& d, int* step_counter) {
  if (p.split_S < 2 || d.n < 1 || d.n > kMaxPeers) return cudaErrorInvalidValue;
  if (ponly_on(p))
    return launch_synthesis_ponly(p, nullptr, p.own_m, p.n_own_m, p.Lp, p.xsynP, xsyn, nb, s,
                                  step_counter, d);
  return synthesis_impl(p, nullptr, p.own_m, p.n_own_m, p.Lp, xsyn, nb, s, step_counter, d);
}

static cudaError_t synthesis_impl(const Plan& p, double2* fsyn, const int* mlist, int nm, int Lp,
                                  const double* xsyn, int nb, cudaStream_t s, int* step_counter,
                                  const SynDst& sd) {
  if (synthesis_bulk_ok(p, nb))  // table-streaming regime (legendre_tma.cu)
    return launch_synthesis_bulk(p, fsyn, mlist, nm, Lp, xsyn, nb, s, step_counter, sd);
  const int NB = pick_nb(nb);
  const int nblk = (nb + NB - 1) / NB;
  // latency regime (few batch blocks): 1 row tile x 4 K-splits (small T) or the
  // plan's WJ x (4 / WJ); throughput regime (many batch blocks): 4 row tiles,
  // no K-split, NBC batch blocks per CTA so the table slice is reused from L1
  int WJ = p.synth_wj, WK = kWarps / WJ, NBC = 1;
  if (nblk >= 4) {
    WJ = (p.J / kRowsPerWarp) % 4 == 0 ? 4 : ((p.J / kRowsPerWarp) % 3 == 0 ? 3 : 2);
    WK = 1;
    NBC = nblk >= 32 ? 8 : (nblk >= 8 ? 4 : 2);
  }
  dim3 grid(p.J / (kRowsPerWarp * WJ), nm, (nblk + NBC - 1) / NBC);
  const dim3 block(32 * WJ * WK);
  // the cp.async pipeline pays off from T255 up, for many batch blocks and at
  // T63; at T127 with few blocks the register-prefetch kernel is faster (measured)
  const bool cp = p.syn_cp >= 0 ? p.syn_cp != 0 : (p.T >= 200 || p.T < 100 || nblk >= 4);
  // prefetch depth 1: a deeper register prefetch costs a resident CTA per SM,
  // which the latency-bound small truncations need more (measured on B200)
#define SDCSW_SYN(NBV)                                                                         \
  if (NB == NBV) {                                                                             \
    if (cp)                                                                                    \
      launch_k(k_synthesis_cp<NBV>, grid, block, syn_cp_smem<NBV>(), s, xsyn, nb, p.T, p.J,    \
               p.ptab_s, p.htab_s, p.rowoff, p.n_even, fsyn, step_counter, WJ, NBC, mlist, Lp, \
               sd);                                                                            \
    else                                                                                       \
    launch_k(k_synthesis<NBV, 1>, grid, block, 0, s, xsyn, nb, p.T, p.J, p.ptab_s, p.htab_s, \
             p.rowoff, p.n_even, fsyn, step_counter, WJ, NBC, mlist, Lp, sd);                  \
    return cudaGetLastError();                                                                 \
  }
  SDCSW_NB_LIST(SDCSW_SYN)
#undef SDCSW_SYN
  return cudaErrorInvalidValue;
}

template <bool FZ>
static cudaError_t analysis_impl(const Plan& p, const Work& w, double2* fe, int nb,
                                 const FuseArgs& fz, cudaStream_t s) {
  const int NB = pick_nb(nb);
  const int* work = p.own_work != nullptr ? p.own_work : p.anal_work;
  const int nwork = p.own_work != nullptr ? p.n_own_work : p.n_anal_work;
  dim3 grid(nwork, (nb + NB - 1) / NB);
  // prefetch depth 1 (see synthesis_impl)
#define SDCSW_ANA(NBV)                                                                          \
  if (NB == NBV) {                                                                              \
    launch_k(k_analysis<NBV, 1, FZ>, grid, 32 * kWarps, 0, s, w.gan, nb, p.T, p.J, p.C, p.ptab_a, \
             p.htab_a, p.rowoff, p.n_even, p.row_n, p.moff, p.lam, work, fe, p.anal_wj, fz,      \
             p.xscale, p.idx_row);                                                              \
    return cudaGetLastError();                                                                  \
  }
  SDCSW_NB_LIST(SDCSW_ANA)
#undef SDCSW_ANA
  return cudaErrorInvalidValue;
}

cudaError_t launch_analysis(const Plan& p, const Work& w, double2* fe, int nb, cudaStream_t s) {
  if (ponly_on(p)) return launch_analysis_ponly(p, w, fe, nb, s);  // P analyses + assembly
  cudaError_t err;
  if (launch_analysis_tma(p, w, fe, nb, s, &err)) return err;  // table-streaming regime
  FuseArgs none{};
  return analysis_impl<false>(p, w, fe, nb, none, s);
}

cudaError_t launch_analysis_fused(const Plan& p, const Work& w, int nb, const FuseArgs& fz,
                                  cudaStream_t s) {
  // one batch block must hold every node (NB = nb), and the epilogue fixes M;
  // publishing (mode 4) handles any batch
  if (fz.mode == 4) {  // (a split plan's analysis computes, and so publishes, own m only)
    if (p.kind != 0 || p.tma_ok || fz.peer_world < 1 ||
        fz.peer_world > kMaxPeers || nb < 1)
      return cudaErrorInvalidValue;
    return analysis_impl<true>(p, w, nullptr, nb, fz, s);
  }
  if (!fuse_supported(p, fz.M) || nb > kFuseMaxNodes || (nb != 1 && nb != fz.M))
    return cudaErrorInvalidValue;
  return analysis_impl<true>(p, w, nullptr, nb, fz, s);
}

}  // namespace sdcsw
