// Ring kernel: per (state, N/S ring pair) inverse longitude FFTs of the four
// synthesised fields, the pointwise nonlinear products on the Gaussian grid
// and the forward FFTs of the five products - all in shared memory, so grid
// data never touches HBM.  Replaces the irfft2 / products / rfft2 chain of the
// planar _f_expl (pkg/src/parsdc/problems/swe.py:176-185) with its spherical
// restatement (A=eta U, B=eta V, C=Phi' U, D=Phi' V,
// E=(U^2+V^2)/(2(1-mu^2))).
//
// FFT: mixed-radix (16, 8, 4, 3) Stockham autosort over nlon = 3*2^k complex
// points (kernel templated on nlon: 96 ... 1536), in place: every pass reads all butterfly inputs of all the
// concurrent transforms into registers, synchronises, then writes.  The two
// real rings of a pair are packed into one complex transform (z = x_N + i x_S),
// and the 4 inverse / 5 forward transforms of a pair run as ONE multi-FFT each,
// so a pair costs 2 * (#radix passes) barrier phases instead of 9x that.
// Output per (b, pair, m <= T): the seven analysis data slots, pre-weighted,
// pre-multiplied by i m where the analysis needs it and folded into symmetric
// (N+S) / antisymmetric (N-S) parts.
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "fft_math.cuh"

#ifndef SDCSW_EXP
#define SDCSW_EXP 0
#endif

#ifndef SDCSW_TW_ALL
#define SDCSW_TW_ALL 1  // multiply by the twiddle at k = 0 too (w^0 = 1): no divergent branch
#endif
namespace sdcsw {
#if SDCSW_EXP == 4
__device__ unsigned long long g_rtimes[1 << 16];
__device__ __forceinline__ unsigned long long gtimer_r() {  // SM cycles (phase differences only)
  return (unsigned long long)clock64();
}
#define RT(i) if (threadIdx.x == 0 && cta < 8192) g_rtimes[8 * cta + (i)] = gtimer_r();
#else
#define RT(i)
#endif

// Shared-memory FFT arrays are padded: element k of a transform lives at
// k + (k >> SH) (SH = 0: unpadded).  Each array generation between two passes
// gets its own SH, chosen at compile time by a bank model of the writing and
// the reading pass (16-byte accesses: a quarter-warp of 8 lanes is one
// 128-byte wavefront when the 8 addresses fall in distinct 16-byte bank groups).
__host__ __device__ constexpr int pzv(int k, int sh) { return sh ? k + (k >> sh) : k; }
template <int N>
constexpr int padded() { return N + N / 8; }  // room for the densest padding (SH = 3)

// Compile-time radix plans.  The inverse plan ends with radix 3 and the
// forward plan (its reverse) starts with it, so the last inverse pass, the
// grid products and the first forward pass run fused in registers on the
// same points (Stockham: the last pass of a plan writes exactly the points
// the first pass of the reversed plan reads).
template <int N> struct RadixPlan;
template <> struct RadixPlan<96> { static constexpr int n = 3; static constexpr int r[6] = {8, 4, 3}; };
template <> struct RadixPlan<192> { static constexpr int n = 3; static constexpr int r[6] = {16, 4, 3}; };
#ifndef SDCSW_PLAN384  // experiment knob; {16, 8, 3} measured best for c1 (round 2)
#define SDCSW_PLAN384 0
#endif
#if SDCSW_PLAN384 == 1
template <> struct RadixPlan<384> { static constexpr int n = 3; static constexpr int r[6] = {8, 16, 3}; };
#elif SDCSW_PLAN384 == 2
template <> struct RadixPlan<384> { static constexpr int n = 4; static constexpr int r[6] = {4, 4, 8, 3}; };
#elif SDCSW_PLAN384 == 3
template <> struct RadixPlan<384> { static constexpr int n = 4; static constexpr int r[6] = {8, 4, 4, 3}; };
#elif SDCSW_PLAN384 == 4
template <> struct RadixPlan<384> { static constexpr int n = 4; static constexpr int r[6] = {4, 8, 4, 3}; };
#else
template <> struct RadixPlan<384> { static constexpr int n = 3; static constexpr int r[6] = {16, 8, 3}; };
#endif
#ifndef SDCSW_PLAN768  // experiment knob
#define SDCSW_PLAN768 0
#endif
#if SDCSW_PLAN768 == 1
template <> struct RadixPlan<768> { static constexpr int n = 4; static constexpr int r[6] = {8, 8, 4, 3}; };
#elif SDCSW_PLAN768 == 2
template <> struct RadixPlan<768> { static constexpr int n = 4; static constexpr int r[6] = {4, 8, 8, 3}; };
#else
template <> struct RadixPlan<768> { static constexpr int n = 3; static constexpr int r[6] = {16, 16, 3}; };
#endif
#ifndef SDCSW_PLAN1536  // experiment knob
#define SDCSW_PLAN1536 0
#endif
#if SDCSW_PLAN1536 == 1
template <> struct RadixPlan<1536> { static constexpr int n = 4; static constexpr int r[6] = {8, 8, 8, 3}; };
#elif SDCSW_PLAN1536 == 2
template <> struct RadixPlan<1536> { static constexpr int n = 4; static constexpr int r[6] = {8, 16, 4, 3}; };
#elif SDCSW_PLAN1536 == 3
template <> struct RadixPlan<1536> { static constexpr int n = 5; static constexpr int r[6] = {8, 4, 4, 4, 3}; };
#else
template <> struct RadixPlan<1536> { static constexpr int n = 4; static constexpr int r[6] = {16, 8, 4, 3}; };
#endif

template <int N>
constexpr int inv_radix(int s) { return RadixPlan<N>::r[s]; }
template <int N>
constexpr int fwd_radix(int s) { return RadixPlan<N>::r[RadixPlan<N>::n - 1 - s]; }
template <int N>
constexpr int inv_prefix(int s) {  // product of the first s inverse radices
  int p = 1;
  for (int q = 0; q < s; ++q) p *= inv_radix<N>(q);
  return p;
}
template <int N>
constexpr int fwd_prefix(int s) {
  int p = 1;
  for (int q = 0; q < s; ++q) p *= fwd_radix<N>(q);
  return p;
}

// ---- bank model ------------------------------------------------------------
// Wavefronts of one 16-byte shared access by lanes it = 0..63 (two warps),
// lane address given in 16-byte units.
template <typename F>
constexpr int wavefronts(F addr) {
  int total = 0;
  for (int ph = 0; ph < 8; ++ph) {  // 8 quarter-warps
    int a[8] = {};
    for (int l = 0; l < 8; ++l) a[l] = addr(ph * 8 + l);
    int worst = 1;
    for (int g = 0; g < 8; ++g) {
      int cnt = 0;
      for (int l = 0; l < 8; ++l) {
        if (a[l] < 0 || ((a[l] % 8) + 8) % 8 != g) continue;
        bool dup = false;
        for (int q = 0; q < l; ++q) dup = dup || a[q] == a[l];
        if (!dup) ++cnt;
      }
      worst = cnt > worst ? cnt : worst;
    }
    total += worst;
  }
  return total;
}
// Stockham pass (R, P) over NF field-major transforms: read of input r, write of output r
template <int N>
constexpr int pass_read_cost(int R, int NF, int sh) {
  int c = 0;
  const int NR = N / R;
  for (int r = 0; r < R; ++r)
    c += wavefronts([&](int it) {
      if (it >= NF * NR) return -1;
      const int f = it / NR, i = it % NR;
      return f * padded<N>() + pzv(i + r * NR, sh);
    });
  return c;
}
template <int N>
constexpr int pass_write_cost(int R, int P, int NF, int sh) {
  int c = 0;
  const int NR = N / R;
  for (int r = 0; r < R; ++r)
    c += wavefronts([&](int it) {
      if (it >= NF * NR) return -1;
      const int f = it / NR, i = it % NR, k = i % P;
      return f * padded<N>() + pzv((i - k) * R + k + r * P, sh);
    });
  return c;
}
// Array generation b (between consecutive passes): inverse passes 0..n-1 (the
// last fused with the products and forward pass 0), forward passes 1..n-1.
// b < n-1: inverse pass b -> inverse pass b+1 (b = n-2: the fused phase reads)
// b = n-1: fused phase (forward pass 0) -> forward pass 1
// b >= n : forward pass b-n+1 -> forward pass b-n+2 (last: the output phase)
template <int N>
constexpr int generation_cost(int b, int sh) {
  constexpr int n = RadixPlan<N>::n;
  int c = 0;
  if (b < n - 1) {
    c += pass_write_cost<N>(inv_radix<N>(b), inv_prefix<N>(b), 4, sh);
    c += pass_read_cost<N>(inv_radix<N>(b + 1), b + 1 == n - 1 ? 1 : 4, sh);
  } else {
    const int s = b - (n - 1);  // forward pass writing this generation
    c += pass_write_cost<N>(fwd_radix<N>(s), fwd_prefix<N>(s), s == 0 ? 1 : 5, sh);
    if (s + 1 < n) c += pass_read_cost<N>(fwd_radix<N>(s + 1), 5, sh);
  }
  return c;
}
template <int N>
constexpr int gen_shift(int b) {
  const int cand[4] = {3, 4, 5, 0};
  int best = cand[0], bc = generation_cost<N>(b, cand[0]);
  for (int q = 1; q < 4; ++q) {
    const int c = generation_cost<N>(b, cand[q]);
    if (c < bc) { bc = c; best = cand[q]; }
  }
  return best;
}

// ---- per-pass twiddle tables -------------------------------------------------
// Pass (R, P) needs w(r, k) = exp(-2 pi i r k / (R P)) for r = 1..R-1, k < P,
// stored at [(r - 1) P + k] so that lanes with consecutive k read consecutive
// entries.  Tables: inverse passes 1..n-1, then forward passes 1..n-1.
template <int N>
constexpr int tw_size_inv(int s) { return (inv_radix<N>(s) - 1) * inv_prefix<N>(s); }
template <int N>
constexpr int tw_size_fwd(int s) { return (fwd_radix<N>(s) - 1) * fwd_prefix<N>(s); }
template <int N>
constexpr int tw_off_inv(int s) {
  int o = 0;
  for (int q = 1; q < s; ++q) o += tw_size_inv<N>(q);
  return o;
}
template <int N>
constexpr int tw_off_fwd(int s) {
  int o = tw_off_inv<N>(RadixPlan<N>::n);
  for (int q = 1; q < s; ++q) o += tw_size_fwd<N>(q);
  return o;
}
template <int N>
constexpr int tw_total() { return tw_off_fwd<N>(RadixPlan<N>::n); }

// Twiddle tables in shared memory (staged per CTA) or read from global
// memory through L1 (saves the staging and shared memory).  Measured on B200:
// global reads win only for the throughput variant at nlon = 384 (128-thread
// CTAs, 5 per SM: 64-member ensemble -6% per step); the latency regime keeps
// 256-thread CTAs with staged twiddles.
template <int N, int THREADS>
constexpr bool ring_twg() { return N == 384 && THREADS == 128; }
template <int N, int THREADS>
constexpr size_t ring_smem_t() {
  return (size_t)(5 * padded<N>() + (ring_twg<N, THREADS>() ? 0 : tw_total<N>())) * sizeof(double2);
}

// One in-place Stockham pass (radix R, sub-length P) over NF concurrent
// transforms of length N at Z[f * padded<N>()], reading generation SHI and
// writing generation SHO; twp = this pass's twiddle table.
// keep >= 0: the plan's last forward pass, whose outputs the output phase reads only at bins
// m <= keep and N - m (the analysis needs m <= T): the other stores are skipped
template <int N, int R, int P, bool INV, int NF, int THREADS, int SHI, int SHO>
__device__ __forceinline__ void pass(double2* Z, const double2* twp, int keep = -1) {
  constexpr int NR = N / R;
  constexpr int ITEMS = NF * NR;
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
      for (int r = 0; r < R; ++r) v[q][r] = X[pzv(i + r * NR, SHI)];
      if (P > 1 && (SDCSW_TW_ALL || k)) {  // (k = 0: the table holds w^0 = 1)
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = twp[(r - 1) * P + k];
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
      for (int r = 0; r < R; ++r) {
        const int bin = jo + r * P;
        if (keep < 0 || bin <= keep || bin >= N - keep) X[pzv(bin, SHO)] = v[q][r];
      }
    }
  }
  __syncthreads();
}

#ifndef SDCSW_RING_P0PAD
#define SDCSW_RING_P0PAD 1  // zero-padded coefficient staging for the first inverse pass
#endif
#ifndef SDCSW_RING_P0DIRECT
#define SDCSW_RING_P0DIRECT 0  // first inverse pass loads its butterfly inputs straight from the
                               // Fourier workspace (no shared-memory staging, two barriers fewer)
#endif
#ifndef SDCSW_RING_PRUNE
#define SDCSW_RING_PRUNE 1  // skip the last forward pass's stores of bins the output never reads
                            // (from nlon 768: T255 ring -1.5%, T511 -0.6%; +0.5% at nlon 384)
#endif
// inverse passes s in [S, n-1) and forward passes s in [S, n)
template <int N, int S, int THREADS>
__device__ __forceinline__ void inverse_mid(double2* Z, const double2* tw) {
  if constexpr (S < RadixPlan<N>::n - 1) {
    pass<N, inv_radix<N>(S), inv_prefix<N>(S), true, 4, THREADS, gen_shift<N>(S - 1),
         gen_shift<N>(S)>(Z, tw + tw_off_inv<N>(S));
    inverse_mid<N, S + 1, THREADS>(Z, tw);
  }
}
template <int N, int S, int THREADS>
__device__ __forceinline__ void forward_rest(double2* Z, const double2* tw, int T) {
  constexpr int n = RadixPlan<N>::n;
  if constexpr (S < n) {
    pass<N, fwd_radix<N>(S), fwd_prefix<N>(S), false, 5, THREADS, gen_shift<N>(n - 2 + S),
         gen_shift<N>(n - 1 + S)>(Z, tw + tw_off_fwd<N>(S),
                                   S == n - 1 && SDCSW_RING_PRUNE && N >= 768 ? T : -1);
    forward_rest<N, S + 1, THREADS>(Z, tw, T);
  }
}

// host: the per-pass twiddle tables gathered from w[k] = exp(-2 pi i k / N)
template <int N>
static void build_pass_twiddles(const double2* w, std::vector<double2>& out) {
  constexpr int n = RadixPlan<N>::n;
  out.assign(tw_total<N>(), make_double2(0.0, 0.0));
  auto fill = [&](int off, int R, int P) {
    const int TS = N / (R * P);
    for (int r = 1; r < R; ++r)
      for (int k = 0; k < P; ++k) out[off + (r - 1) * P + k] = w[r * k * TS];
  };
  for (int s = 1; s < n; ++s) fill(tw_off_inv<N>(s), inv_radix<N>(s), inv_prefix<N>(s));
  for (int s = 1; s < n; ++s) fill(tw_off_fwd<N>(s), fwd_radix<N>(s), fwd_prefix<N>(s));
}

#ifndef SDCSW_RING_MINB128
#define SDCSW_RING_MINB128 5  // 96 registers: 5 CTAs per SM (throughput variant)
#endif
#ifndef SDCSW_RING_MINB768
#define SDCSW_RING_MINB768 2  // shared memory allows 2 CTAs per SM anyway: up to 128 registers (T255 -2%)
#endif
template <int N, int THREADS>
constexpr int ring_min_blocks() {
  return N == 768 ? SDCSW_RING_MINB768
                  : (THREADS <= 128 ? SDCSW_RING_MINB128 : (THREADS <= 256 ? 3 : 1));
}

#ifndef SDCSW_RING_L2PF
#define SDCSW_RING_L2PF 1536  // nlon from which the ring kernel prefetches one wave ahead
#endif
// resident CTAs per SM of a ring kernel (shared memory bound; registers allow more)
template <int N, int THREADS>
constexpr int ring_resident() {
  return (int)(232448 / (ring_smem_t<N, THREADS>() + 1024)) < ring_min_blocks<N, THREADS>()
             ? (int)(232448 / (ring_smem_t<N, THREADS>() + 1024))
             : ring_min_blocks<N, THREADS>();
}

// Output stores of the ring kernel: the analysis data of one latitude pair is
// a column of the [state][m][j] layout (224 bytes per m, strided by J x 224),
// so the CTA stages its values in shared memory (the dead FFT arrays) and one
// thread writes them with TMA tensor stores (box rows = wavenumbers), instead
// of 16-byte stores from every thread.
struct alignas(64) GanMaps {
  CUtensorMap rec;  // record order: {28 doubles, J, rows}
  CUtensorMap fp;   // fragment order, P part: {8 doubles, j & 3, fold, j >> 2, rows}
  CUtensorMap fh;   // fragment order, H part: {6 doubles, j & 3, fold, j >> 2, rows}
  CUtensorMap f5;   // H-free path (po): {10 doubles, j & 3, fold, j >> 2, rows}
  int rows;         // wavenumbers per store box (divides L); 0 = plain stores
  int row0;         // first row of the launch's workspace (batch offset x L)
  int po;           // 1: write the five-slot data of the H-free analysis (ganp_off)
};

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
          reinterpret_cast<unsigned long long>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(src))
      : "memory");
}

template <int N, int THREADS, bool SPLIT>
__global__ void __launch_bounds__(THREADS, ring_min_blocks<N, THREADS>()) k_ring(const double2* __restrict__ fsyn,
                                                  double2* __restrict__ gan, int J, int T,
                                                  const double* __restrict__ mu,
                                                  const double* __restrict__ wsyn,
                                                  const double* __restrict__ wke,
                                                  const double2* __restrict__ twg,
                                                  double two_omega,
                                                  const int* __restrict__ m_part,
                                                  const int* __restrict__ m_k, int Lp, int nbg,
                                                  int frag, const RingPeer rp,
                                                  const __grid_constant__ GanMaps gm) {
  SDCSW_PDL_ENTRY();
  if (SDCSW_TRIG_RING == 1) SDCSW_PDL_TRIGGER();
  extern __shared__ __align__(128) double2 sm2[];
  constexpr int NP = padded<N>();
  constexpr int NS = RadixPlan<N>::n;
  constexpr int TWN = tw_total<N>();
  double2* Z = sm2;             // [5][NP] (padded)
  constexpr bool TWG = ring_twg<N, THREADS>();
  // per-pass twiddle tables: global (read through L1) or staged in shared memory
  const double2* tw = TWG ? twg : sm2 + 5 * NP;
  const int L = T + 1;
  const int j = blockIdx.x, b = blockIdx.y;
  // Fourier coefficients of (b, j, m): part-major [part][nbg][J][Lp][4 fields][2 (N, S)]
  // (unsplit: one part, k = m, Lp = L)
  const double2* F0 = fsyn + ((size_t)b * J + j) * Lp * 8;  // unsplit: part 0, k = m
  auto Fm = [&](int m) -> const double2* {
    if constexpr (!SPLIT) {
      return F0 + (size_t)m * 8;
    } else {
      const int part = m_part[m], k = m_k[m];
      return fsyn + ((((size_t)part * nbg + b) * J + j) * Lp + k) * 8;
    }
  };
#if SDCSW_EXP == 4
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
#endif
  RT(0)
  // constant plan data before the dependency wait (overlaps the producer's
  // tail): the twiddle tables arrive by one asynchronous bulk copy, waited for
  // only before the first pass that uses them (pass 0 has none)
  __shared__ __align__(8) unsigned long long twbar;
  if constexpr (!TWG) {
    if (threadIdx.x == 0) {
      mbar_init(&twbar, 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&twbar, (unsigned)(TWN * sizeof(double2)));
      bulk_g2s(sm2 + 5 * NP, twg, (unsigned)(TWN * sizeof(double2)), &twbar);
    }
  }
  const double muj = mu[j], ws = wsyn[j], wk = wke[j];
  RT(6)
  SDCSW_PDL_WAIT();
  if constexpr (!SPLIT && N >= SDCSW_RING_L2PF) {
    // many waves (large nlon): pull the Fourier block of the CTA one wave ahead
    // (linear index + resident CTAs) into L2, so its load phase hits L2 (T511, 5 states:
    // 296.7 -> 290.0 us; neutral at nlon 768, measured)
    if (threadIdx.x == 0) {
      unsigned nsm;
      asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
      const unsigned ahead = nsm * (unsigned)ring_resident<N, THREADS>();
      const unsigned nxt = blockIdx.y * gridDim.x + blockIdx.x + ahead;
      if (nxt < gridDim.x * gridDim.y) {
        const double2* src = fsyn + (size_t)nxt * Lp * 8;  // [b][j] blocks are consecutive
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src),
                     "r"((unsigned)(Lp * 8 * sizeof(double2)))
                     : "memory");
      }
    }
  }
  unsigned long long fx = 0;  // spectral split over peer memory: Fourier exchange number
  if constexpr (SPLIT) {
    if (rp.flags != nullptr) {
      fx = *reinterpret_cast<volatile unsigned long long*>(rp.fseq) + 1;
      if (threadIdx.x == 0) {  // post own part (written by the completed synthesis), wait for all
        if (rp.world > 1) __threadfence_system();
        for (int q = 0; q < rp.world; ++q) atomicMax_system(rp.post[q], fx);
        for (int q = 0; q < rp.world; ++q)
          if (!wait_posted(&rp.flags->flag[q], fx, rp.to, q, 1)) break;
      }
      __syncthreads();
      fsyn += (fx & 1) * rp.par_stride;
    }
  }

  // ---- inverse pass 0 (P = 1, no twiddles) from the Fourier coefficients:
  //      Z_m = X_m + i Y_m, Z_{N-m} = conj(X_m) + i conj(Y_m).
  //      The coefficients are first staged (coalesced, all loads in flight)
  //      into the Z area as Fs[hemisphere][field][m] (row stride L + 1); the
  //      pass then reads them, syncs and writes its outputs over them (the
  //      in-place Stockham pattern).
  {
    constexpr int R = inv_radix<N>(0);
    constexpr int NR = N / R;
    constexpr int ITEMS = 4 * NR;
    constexpr int MAXIT = (ITEMS + THREADS - 1) / THREADS;
    constexpr int SHO = gen_shift<N>(0);
    double2* Fs = Z;
    // zero-padded rows (m = L..N/2 hold zeros): the pass reads bin min(k, N - k) for every
    // k without a branch on the truncation (SDCSW_RING_P0PAD=0: rows of L, masked reads)
    constexpr int LP = SDCSW_RING_P0PAD ? N / 2 + 1 : 0;
    const int LS = SDCSW_RING_P0PAD ? LP : L + 1;
    if constexpr (!SDCSW_RING_P0DIRECT) {
      for (int e = threadIdx.x; e < 8 * L; e += THREADS) {  // coalesced
        const int m = e >> 3, fh = e & 7;  // fh = 2 field + hemisphere
        Fs[((fh & 1) * 4 + (fh >> 1)) * LS + m] = Fm(m)[fh];
      }
      if (SDCSW_RING_P0PAD)
        for (int e = threadIdx.x; e < 8 * (LP - L); e += THREADS) {
          const int row = e / (LP - L), m = L + (e - row * (LP - L));
          Fs[row * LS + m] = make_double2(0.0, 0.0);
        }
      __syncthreads();
    }
    RT(7)
    double2 v[MAXIT][R];
#pragma unroll
    for (int q = 0; q < MAXIT; ++q) {
      const int it = threadIdx.x + q * THREADS;
      if (ITEMS % THREADS == 0 || it < ITEMS) {
        const int f = it / NR, i = it - f * NR;
        const double2* FN = Fs + f * LS;
        const double2* FS = Fs + (4 + f) * LS;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int k = i + r * NR;
          bool lo;
          double2 xn, xs;
          if constexpr (SDCSW_RING_P0DIRECT) {
            // (field f, m): the N and S values are one 32-byte record of the workspace
            lo = k <= N / 2;
            const int mm = lo ? k : N - k;
            xn = make_double2(0.0, 0.0);
            xs = xn;
            if (mm <= T) {
              const double2* src = Fm(mm) + 2 * f;
              xn = src[0];
              xs = src[1];
            }
          } else if constexpr (SDCSW_RING_P0PAD) {
            lo = k <= N / 2;
            const int mm = lo ? k : N - k;
            xn = FN[mm];
            xs = FS[mm];
          } else {
            lo = k <= T;
            const bool hi = k >= N - T;
            xn = make_double2(0.0, 0.0);
            xs = xn;
            if (lo || hi) {
              const int mm = lo ? k : N - k;
              xn = FN[mm];
              xs = FS[mm];
            }
          }
          if (k == 0) xn.y = xs.y = 0.0;
          v[q][r] = lo ? make_double2(xn.x - xs.y, xn.y + xs.x)
                       : make_double2(xn.x + xs.y, xs.x - xn.y);
        }
        dft<R, true>(v[q]);
      }
    }
    if constexpr (!SDCSW_RING_P0DIRECT) __syncthreads();  // (staged inputs read in place)
#pragma unroll
    for (int q = 0; q < MAXIT; ++q) {
      const int it = threadIdx.x + q * THREADS;
      if (ITEMS % THREADS == 0 || it < ITEMS) {
        const int f = it / NR, i = it - f * NR;
        double2* X = Z + f * NP;
#pragma unroll
        for (int r = 0; r < R; ++r) X[pzv(i * R + r, SHO)] = v[q][r];
      }
    }
    __syncthreads();
  }
  RT(1)
  if constexpr (!TWG) mbar_wait(&twbar, 0);  // (the staging barrier above ordered the init)
  inverse_mid<N, 1, THREADS>(Z, tw);
  RT(2)

  // ---- fused: last inverse pass (radix 3, P = N/3), grid products, first
  //      forward pass (radix 3, P = 1) on the points i + r N/3
  {
    constexpr int N3 = N / 3;
    constexpr int SHI = gen_shift<N>(NS - 2), SHO = gen_shift<N>(NS - 1);
    static_assert(inv_prefix<N>(NS - 1) == N3, "inverse plan must end with radix 3");
    static_assert(inv_radix<N>(NS - 1) == 3, "inverse plan must end with radix 3");
    const double2* twp = tw + tw_off_inv<N>(NS - 1);
    const double cor_n = two_omega * muj, cor_s = -two_omega * muj;
    const double ke_scale = 0.5 / ((1.0 - muj) * (1.0 + muj));
    constexpr int MAXIT = (N3 + THREADS - 1) / THREADS;
    double2 out[MAXIT][5][3];
#pragma unroll
    for (int q = 0; q < MAXIT; ++q) {
      const int i = threadIdx.x + q * THREADS;
      if (N3 % THREADS == 0 || i < N3) {
        double2 g[4][3];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const double2* X = Z + f * NP;
#pragma unroll
          for (int r = 0; r < 3; ++r) g[f][r] = X[pzv(i + r * N3, SHI)];
          if (SDCSW_TW_ALL || i) {  // twiddles exp(+2 pi i r i / N) (i = 0: 1)
#pragma unroll
            for (int r = 1; r < 3; ++r) {
              double2 w = twp[(r - 1) * N3 + i];
              w.y = -w.y;
              g[f][r] = cmul(g[f][r], w);
            }
          }
          dft<3, true>(g[f]);
        }
        // products at the three points (re = north ring, im = south ring)
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double2 U = g[0][r], V = g[1][r], Zt = g[2][r], Ph = g[3][r];
          const double en = Zt.x + cor_n, es = Zt.y + cor_s;
          out[q][0][r] = make_double2(en * U.x, es * U.y);   // A = eta U
          out[q][1][r] = make_double2(en * V.x, es * V.y);   // B = eta V
          out[q][2][r] = make_double2(Ph.x * U.x, Ph.y * U.y);  // C = Phi U
          out[q][3][r] = make_double2(Ph.x * V.x, Ph.y * V.y);  // D = Phi V
          out[q][4][r] = make_double2((U.x * U.x + V.x * V.x) * ke_scale,
                                      (U.y * U.y + V.y * V.y) * ke_scale);  // kinetic energy
        }
#pragma unroll
        for (int o = 0; o < 5; ++o) dft<3, false>(out[q][o]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < MAXIT; ++q) {
      const int i = threadIdx.x + q * THREADS;
      if (N3 % THREADS == 0 || i < N3) {
#pragma unroll
        for (int o = 0; o < 5; ++o)
#pragma unroll
          for (int r = 0; r < 3; ++r) Z[o * NP + pzv(3 * i + r, SHO)] = out[q][o][r];
      }
    }
    __syncthreads();
  }
  RT(3)
  forward_rest<N, 1, THREADS>(Z, tw, T);
  if (SDCSW_TRIG_RING == 2) SDCSW_PDL_TRIGGER();
  RT(4)

  const double h = 0.5 / (double)N;
  constexpr int SHL = gen_shift<N>(2 * NS - 2);
  // the seven analysis data slots (internal.cuh order) of item (m, fold)
  auto item = [&](int it, double2 (&o)[kNumSlots]) {
    const int m = it >> 1, fold = it & 1;
    const double dm = (double)m;
    double2 v[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double2 zm = Z[q * NP + pzv(m, SHL)], zc = Z[q * NP + pzv(m == 0 ? 0 : N - m, SHL)];
      // X = FFT(north)/N, Y = FFT(south)/N; fold 0: S = X + Y, fold 1: A = X - Y
      const double2 X = make_double2(h * (zm.x + zc.x), h * (zm.y - zc.y));
      const double2 Y = make_double2(h * (zm.y + zc.y), -h * (zm.x - zc.x));
      v[q] = fold ? csub(X, Y) : cadd(X, Y);
    }
    // A = eta U: X_zeta = -(i m A) ws, Y_delta = A ws; B = eta V: X_delta = (i m B) ws,
    // Y_zeta = B ws; C = Phi U: X_phi = -(i m C) ws; D = Phi V: Y_phi = D ws; X_ke = E wk
    o[kXPhi] = make_double2(dm * v[2].y * ws, -dm * v[2].x * ws);
    o[kXZeta] = make_double2(dm * v[0].y * ws, -dm * v[0].x * ws);
    o[kXDelta] = make_double2(-dm * v[1].y * ws, dm * v[1].x * ws);
    o[kXKe] = make_double2(v[4].x * wk, v[4].y * wk);
    o[kYPhi] = make_double2(v[3].x * ws, v[3].y * ws);
    o[kYZeta] = make_double2(v[1].x * ws, v[1].y * ws);
    o[kYDelta] = make_double2(v[0].x * ws, v[0].y * ws);
  };
  constexpr int MI = (2 * ((N + 2) / 3) + THREADS - 1) / THREADS;  // items per thread, L <= (N + 2) / 3
  // H-free path: the five products of item (m, fold), folded and weighted (A..D by
  // w_s, E by w_ke); the i m factors and the recurrence act after the analysis
  auto item5 = [&](int it, double2 (&o)[kSlotsP]) {
    const int m = it >> 1, fold = it & 1;
#pragma unroll
    for (int q = 0; q < kSlotsP; ++q) {
      const double2 zm = Z[q * NP + pzv(m, SHL)], zc = Z[q * NP + pzv(m == 0 ? 0 : N - m, SHL)];
      const double2 X = make_double2(h * (zm.x + zc.x), h * (zm.y - zc.y));
      const double2 Y = make_double2(h * (zm.y + zc.y), -h * (zm.x - zc.x));
      const double2 v = fold ? csub(X, Y) : cadd(X, Y);
      const double wq = q == 4 ? wk : ws;
      o[q] = make_double2(v.x * wq, v.y * wq);
    }
  };
  if (gm.po) {
    if (gm.rows > 0 && L <= (N + 2) / 3) {  // staged as [m][fold][5 slots], TMA stores
      double2 o[MI][kSlotsP];
#pragma unroll
      for (int q = 0; q < MI; ++q) {
        const int it = threadIdx.x + q * THREADS;
        if (it < 2 * L) item5(it, o[q]);
      }
      __syncthreads();  // every read of the FFT arrays is done
#pragma unroll
      for (int q = 0; q < MI; ++q) {
        const int it = threadIdx.x + q * THREADS;
        if (it < 2 * L) {
#pragma unroll
          for (int k = 0; k < kSlotsP; ++k) Z[it * kSlotsP + k] = o[q][k];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        const int row = gm.row0 + b * L;
        for (int m0 = 0; m0 < L; m0 += gm.rows)
          tma_store_5d(&gm.f5, Z + m0 * 2 * kSlotsP, 0, j & 3, 0, j >> 2, row + m0);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
      double* outp = reinterpret_cast<double*>(gan) + (size_t)b * L * J * kGanP;
      for (int it = threadIdx.x; it < 2 * L; it += THREADS) {
        double2 o[kSlotsP];
        item5(it, o);
        double2* d = reinterpret_cast<double2*>(outp + (size_t)(it >> 1) * J * kGanP +
                                                ganp_off(j, it & 1, 0, 0));
#pragma unroll
        for (int k = 0; k < kSlotsP; ++k) d[k] = o[k];
      }
    }
  } else if (gm.rows > 0 && L <= (N + 2) / 3) {  // (then the boxes fit in the 5 FFT arrays)
    // staged in the FFT arrays as the store boxes: record order [m][fold][7 slots];
    // fragment order [m][fold][4 P slots] then, from L x 128 bytes, [m][fold][3 H slots]
    double2 o[MI][kNumSlots];
#pragma unroll
    for (int q = 0; q < MI; ++q) {
      const int it = threadIdx.x + q * THREADS;
      if (it < 2 * L) item(it, o[q]);
    }
    __syncthreads();  // every read of the FFT arrays is done
    double2* st = Z;
#pragma unroll
    for (int q = 0; q < MI; ++q) {
      const int it = threadIdx.x + q * THREADS;
      if (it < 2 * L) {
        if (!frag) {
#pragma unroll
          for (int k = 0; k < kNumSlots; ++k) st[it * kNumSlots + k] = o[q][k];
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) st[it * 4 + k] = o[q][k];
#pragma unroll
          for (int k = 0; k < 3; ++k) st[8 * L + it * 3 + k] = o[q][4 + k];
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const int row = gm.row0 + b * L;
      for (int m0 = 0; m0 < L; m0 += gm.rows) {
        if (!frag) {
          tma_store_3d(&gm.rec, st + m0 * 2 * kNumSlots, 0, j, row + m0);
        } else {
          tma_store_5d(&gm.fp, st + m0 * 8, 0, j & 3, 0, j >> 2, row + m0);
          tma_store_5d(&gm.fh, st + 8 * L + m0 * 6, 0, j & 3, 0, j >> 2, row + m0);
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // before the CTA exits
    }
  } else {
    // record order - thread (m, fold) writes the fold's seven slots (112
    // contiguous bytes); fragment order (frag, TMA analysis) - the four P
    // slots (64 bytes) and three H slots (48 bytes)
    double* outp = reinterpret_cast<double*>(gan) + (size_t)b * L * J * 28;
    const int pofs = frag ? gan_off(j, 0, kXPhi, 0) : j * 28;
    const int hofs = frag ? gan_off(j, 0, kYPhi, 0) : j * 28 + 2 * kYPhi;
    const int fstride = frag ? 56 : 14;
    for (int it = threadIdx.x; it < 2 * L; it += THREADS) {
      double2 o[kNumSlots];
      item(it, o);
      double* bm = outp + (size_t)(it >> 1) * J * 28 + (it & 1) * fstride;
      double2* dp = reinterpret_cast<double2*>(bm + pofs);  // X_phi, X_zeta, X_delta, X_ke
      double2* dh = reinterpret_cast<double2*>(bm + hofs);  // Y_phi, Y_zeta, Y_delta
#pragma unroll
      for (int k = 0; k < 4; ++k) dp[k] = o[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) dh[k] = o[4 + k];
    }
  }
  if constexpr (SPLIT) {
    if (rp.flags != nullptr) {  // the last CTA to finish completes exchange fx for this rank
      __syncthreads();
      if (threadIdx.x == 0 &&
          atomicAdd(rp.done, 1u) == gridDim.x * gridDim.y - 1) {
        *rp.done = 0;
        *rp.fseq = fx;
      }
    }
  }
#if SDCSW_EXP == 4
  __syncthreads();
#endif
  RT(5)
}

#ifndef SDCSW_RT96
#define SDCSW_RT96 256
#endif
#ifndef SDCSW_RT192
#define SDCSW_RT192 256
#endif
#ifndef SDCSW_RT384
#define SDCSW_RT384 256
#endif
#ifndef SDCSW_RT768
#define SDCSW_RT768 256
#endif
#ifndef SDCSW_RT1536
#define SDCSW_RT1536 512
#endif
#define SDCSW_RING_SIZES(X) \
  X(96, SDCSW_RT96) X(192, SDCSW_RT192) X(384, SDCSW_RT384) X(768, SDCSW_RT768) X(1536, SDCSW_RT1536)
// throughput variants (batches of at least kRingTputBatch states)
#define SDCSW_RING_TPUT(X) X(384, 128)
constexpr int kRingTputBatch = 16;

bool ring_supported(int nlon) {
#define SDCSW_RING_OK(NV, TV) if (nlon == NV) return true;
  SDCSW_RING_SIZES(SDCSW_RING_OK)
#undef SDCSW_RING_OK
  return false;
}

size_t ring_smem_bytes(int nlon);

// Each ring kernel's dynamic shared-memory limit is its own size's need (a
// process-wide function attribute: it must not depend on which plan set it).
cudaError_t configure_ring(size_t /*smem*/) {
  cudaError_t e = cudaSuccess;
#define SDCSW_RING_CFG(NV, TV)                                                                     \
  if (e == cudaSuccess)                                                                            \
    e = cudaFuncSetAttribute(k_ring<NV, TV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                             (int)ring_smem_t<NV, TV>());                                          \
  if (e == cudaSuccess)                                                                            \
    e = cudaFuncSetAttribute(k_ring<NV, TV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             (int)ring_smem_t<NV, TV>());
  SDCSW_RING_SIZES(SDCSW_RING_CFG)
  SDCSW_RING_TPUT(SDCSW_RING_CFG)
#undef SDCSW_RING_CFG
  return e;
}

#if SDCSW_EXP == 4
extern "C" int sdcsw_debug_rtimes(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_rtimes, n * sizeof(unsigned long long));
}
#endif

size_t ring_smem_bytes(int nlon) {
#define SDCSW_RING_SMEM(NV, TV) \
  if (nlon == NV) return ring_smem_t<NV, TV>();
  SDCSW_RING_SIZES(SDCSW_RING_SMEM)
#undef SDCSW_RING_SMEM
  return 0;
}

// per-pass twiddle tables of the ring FFT plan for nlon, from w[k] = exp(-2 pi i k / nlon)
bool ring_pass_twiddles(int nlon, const double2* w, std::vector<double2>& out) {
#define SDCSW_RING_TW(NV, TV) \
  if (nlon == NV) { build_pass_twiddles<NV>(w, out); return true; }
  SDCSW_RING_SIZES(SDCSW_RING_TW)
#undef SDCSW_RING_TW
  return false;
}

// Store maps over the whole analysis workspace (rows = max_batch x L).
// Box rows: L up to 256, else the largest multiple of 4 dividing L up to 256
// (box offsets in shared memory stay 128-byte aligned); none: plain stores.
cudaError_t make_gan_maps(Plan& p) {
  p.gmap_rows = 0;
  p.gmap_frag = false;
  const char* env = getenv("SDCSW_RING_TMA_STORE");
  if (env != nullptr && atoi(env) == 0) return cudaSuccess;
  const int L = p.L, J = p.J;
  int rows = L <= 256 ? L : 0;
  for (int r = 256; rows == 0 && r >= 4; r -= 4)
    if (L % r == 0) rows = r;
  if (rows == 0) return cudaSuccess;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn || q != cudaDriverEntryPointSuccess) return cudaSuccess;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  const cuuint64_t R = (cuuint64_t)p.max_batch * L, rs = (cuuint64_t)J * 28 * sizeof(double);
  auto enc = [&](int i, void* base, cuuint32_t rank, const cuuint64_t* dims, const cuuint64_t* strides,
                 const cuuint32_t* box) {
    const cuuint32_t elem[5] = {1, 1, 1, 1, 1};
    return encode(reinterpret_cast<CUtensorMap*>(&p.gmap[i]), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, base,
                  dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  {
    const cuuint64_t dims[3] = {28, (cuuint64_t)J, R}, strides[2] = {28 * sizeof(double), rs};
    const cuuint32_t box[3] = {28, 1, (cuuint32_t)rows};
    if (!enc(0, p.gan, 3, dims, strides, box)) return cudaSuccess;
  }
  p.gmap_rows = rows;
  if (J % 4 == 0) {  // fragment order (gan_off): [j >> 2][fold][P: j & 3 x 8 | H: j & 3 x 6]
    const cuuint64_t dp[5] = {8, 4, 2, (cuuint64_t)J / 4, R}, dh[5] = {6, 4, 2, (cuuint64_t)J / 4, R};
    const cuuint64_t sp[4] = {64, 448, 896, rs}, sh[4] = {48, 448, 896, rs};
    const cuuint32_t bp[5] = {8, 1, 2, 1, (cuuint32_t)rows}, bh[5] = {6, 1, 2, 1, (cuuint32_t)rows};
    p.gmap_frag = enc(1, p.gan, 5, dp, sp, bp) &&
                  enc(2, reinterpret_cast<double*>(p.gan) + 32, 5, dh, sh, bh);
  }
  p.gmapP_rows = 0;
  if (J % 4 == 0) {  // H-free five-slot data (ganp_off): [j >> 2][fold][j & 3][10]
    const cuuint64_t d5[5] = {10, 4, 2, (cuuint64_t)J / 4, R};
    const cuuint64_t s5[4] = {80, 320, 640, (cuuint64_t)J * 20 * sizeof(double)};
    const cuuint32_t b5[5] = {10, 1, 2, 1, (cuuint32_t)rows};
    const cuuint32_t elem[5] = {1, 1, 1, 1, 1};
    if (encode(reinterpret_cast<CUtensorMap*>(p.gmapP), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, p.gan, d5,
               s5, b5, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      p.gmapP_rows = rows;
  }
  return cudaSuccess;
}

static cudaError_t ring_impl(const Plan& p, const double2* fsyn, double2* gan, const int* m_part,
                             const int* m_k, int Lp, int nb, cudaStream_t s,
                             const RingPeer& rp = RingPeer{}) {
  dim3 grid(p.J, nb);
  const int po = (int)ponly_on(p);  // five-slot output for the H-free analysis
  const int frag = (int)tma_active(p);
  GanMaps gm;
  std::memcpy(&gm.rec, p.gmap[0], sizeof(CUtensorMap));
  std::memcpy(&gm.fp, p.gmap[1], sizeof(CUtensorMap));
  std::memcpy(&gm.fh, p.gmap[2], sizeof(CUtensorMap));
  std::memcpy(&gm.f5, p.gmapP, sizeof(CUtensorMap));
  gm.po = po;
  gm.rows = po ? p.gmapP_rows : (frag && !p.gmap_frag ? 0 : p.gmap_rows);
  gm.row0 = (int)((gan - p.gan) / ((size_t)p.J * p.L * (po ? kSlotsP : kNumSlots) * 2)) * p.L;
#define SDCSW_RING_LAUNCH(NV, TV)                                                                  \
  if (p.nlon == NV) {                                                                              \
    constexpr size_t smem = ring_smem_t<NV, TV>();                                                 \
    if (m_part != nullptr)                                                                         \
      launch_k(k_ring<NV, TV, true>, grid, TV, smem, s, fsyn, gan, p.J, p.T, p.mu, p.wsyn,        \
               p.wke, p.twiddle, 2.0 * p.omega, m_part, m_k, Lp, nb, frag, rp, gm);             \
    else                                                                                           \
      launch_k(k_ring<NV, TV, false>, grid, TV, smem, s, fsyn, gan, p.J, p.T, p.mu, p.wsyn,       \
               p.wke, p.twiddle, 2.0 * p.omega, m_part, m_k, Lp, nb, frag, rp, gm);             \
    return cudaGetLastError();                                                                     \
  }
  if (nb >= kRingTputBatch) {
    SDCSW_RING_TPUT(SDCSW_RING_LAUNCH)
  }
  SDCSW_RING_SIZES(SDCSW_RING_LAUNCH)
#undef SDCSW_RING_LAUNCH
  return cudaErrorInvalidValue;
}

cudaError_t launch_ring(const Plan& p, const Work& w, int nb, cudaStream_t s) {
  // workspace Fourier buffers are unsplit ([nb][J][L][4][2]; part 0, k = m)
  return ring_impl(p, w.fsyn, w.gan, nullptr, nullptr, p.T + 1, nb, s);
}

cudaError_t launch_ring_split(const Plan& p, const Work& w, int nb, cudaStream_t s) {
  return ring_impl(p, p.fsyn_ext, w.gan, p.m_part, p.m_k, p.Lp, nb, s);
}

cudaError_t launch_ring_peer(const Plan& p, const Work& w, const double2* fbase, int nb,
                             cudaStream_t s, const RingPeer& rp) {
  if (p.split_S < 2 || rp.flags == nullptr || rp.world < 1 || rp.world > kMaxPeers)
    return cudaErrorInvalidValue;
  return ring_impl(p, fbase, w.gan, p.m_part, p.m_k, p.Lp, nb, s, rp);
}

}  // namespace sdcsw
