// Internal declarations shared by the libsdcsw.so translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/sdcsw.h"

namespace sdcsw {

// Warp tile of the Legendre GEMMs: two m8 row tiles (16 rows) per warp.
constexpr int kRowsPerWarp = 16;
// Rows of the synthesis K-loop staged in shared memory per chunk.
constexpr int kSynthChunk = 32;
// Latitudes of the analysis K-loop staged per chunk.
constexpr int kAnalChunk = 32;
// Parity-sorted table rows are padded to a multiple of this (an m8 tile is
// then always of a single parity class).
constexpr int kRowPad = 8;

// Analysis data slots written by the ring kernel per (batch, pair, m):
// P-data: X_phi, X_zeta, X_delta, X_ke; H-data: Y_phi, Y_zeta, Y_delta.
enum { kXPhi = 0, kXZeta, kXDelta, kXKe, kYPhi, kYZeta, kYDelta, kNumSlots };

// Analysis data layouts of one (state b, wavenumber m) block of J x 28 doubles.
// Record order (k_analysis, latency regime): [j][fold S, A][7 slots][re, im].
// Fragment order (k_analysis_tma, table-streaming regime; gan_off): per k-step
// of 4 latitudes and fold, [P part: 4 lat x slots 0-3 x (re, im) = 32][H part:
// 4 lat x slots 4-6 x (re, im) = 24], so that one DMMA B fragment (the 8 P
// columns or 6 H columns of one state) is 32 (24) consecutive doubles.
// (Measured: fragment order speeds the TMA analysis up by 20% at T511 and
// slows the latency-regime analysis at T127-T255.)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int gan_off(int j, int fold, int slot, int ri) {
  const int base = ((j >> 2) * 2 + fold) * 56, t = j & 3;
  return slot < 4 ? base + t * 8 + slot * 2 + ri : base + 32 + t * 6 + (slot - 4) * 2 + ri;
}

struct FftPlan {
  int n;           // nlon
  int nstages;     // number of radix passes
  int radix[16];   // radices in application order
};

struct Plan {
  int kind;      // 0: spherical (Legendre + ring FFTs); 1: planar doubly periodic (2-D FFTs)
  int device;
  int T, nlat, nlon, J, C, L;  // L = T+1 (Fourier modes kept)
  int max_batch;
  int rows;                    // packed table rows
  double radius, omega, phibar;
  // device constants
  double* ptab;     // [rows][J] (the TMA analysis streams this layout)
  double* htab;     // [rows][J]
  // the same tables in DMMA-fragment order: one warp's A fragment (8 x 4 for
  // the analysis, 4 x 8 for the synthesis) is 32 consecutive doubles
  double* ptab_a;   // [rows/8][J/4][8 rows][4 lats]
  double* htab_a;
  double* ptab_s;   // [rows/4][J/8][8 lats][4 rows] (lane order g * 4 + t)
  double* htab_s;
  int* rowoff;      // [T+2]
  int* n_even;      // [T+1]
  int* row_n;       // [rows]
  int* moff;        // [T+2] triangular offsets
  double* lam;      // [C]
  double* inv_nn;   // [C] 1/(n(n+1)), 0 for n = 0
  double2* xscale;  // [C] (m a / (n(n+1)), a / (n(n+1))): synthesis B-operand scales
  int* idx_row;     // [C] absolute packed table row of coefficient idx
  double* mu;       // [J] northern nodes
  double* wsyn;     // [J] 2 pi w_j / (a (1 - mu_j^2))
  double* wke;      // [J] 2 pi w_j
  double2* twiddle; // ring FFT per-pass twiddle tables (ring_pass_twiddles)
  int* anal_work;   // [n_anal_work] (m << 16 | row block of anal_wj tiles)
  int n_anal_work;
  int* anal_work4;  // [n_anal_work4] row blocks of 4 tiles (throughput regime)
  int n_anal_work4;
  int synth_wj, anal_wj;  // row tiles per CTA (the other warps split K)
  int syn_cp;             // synthesis with the cp.async pipeline: 1 / 0 / -1 = automatic
  double* resid_part;     // residual partials (lazily allocated, sdcsw_sweep_nodes_residual)
  unsigned* resid_count;
  int ana_nb;             // cap on states per table-streaming analysis CTA (0: all, up to 6)
  int ana_bulk;           // table-streaming analysis with the B operand staged: 1 (default) / 0
  int syn_bulk;           // CTA-staged bulk-copy synthesis (T >= 400): 1 / 0 / -1 = automatic
  FftPlan fft;
  // workspaces
  double2* fsyn;    // [max_batch][J][L][4 fields][2 (N, S)]
  double2* gan;     // [max_batch][L][J][2 (S,A)][kNumSlots]  (GEMM-ready for the analysis)
  double* coef_dev; // small per-call coefficient staging [kCoefCap]
  double* xsyn;     // [rows][max_batch][12] synthesis B operand for API calls
  int xsyn_nb;      // record batch of the last API prep (padding rows zero for it)
  int fe_chunk;     // f_E batch chunk keeping the Fourier workspaces L2-resident (0 = no chunking)
  int ring_threads;
  bool ensemble;    // max_batch >= kEnsembleBatch: throughput-regime kernel choices
  size_t ring_smem;
  // TMA tensor maps (CUtensorMap, 128 B each) over the P / H tables for the
  // table-streaming analysis (T >= 400); tma_ok = maps built
  alignas(64) unsigned long long tmap[2][16];
  bool tma_ok;
  // TMA tensor maps over the analysis data for the ring kernel's output
  // stores (ring_fft.cu): record order, fragment-order P part, H part;
  // gmap_rows = rows (wavenumbers) per store box, 0 = plain stores
  alignas(64) unsigned long long gmap[3][16];
  int gmap_rows;
  bool gmap_frag;  // the fragment-order maps were built
  // spectral split: the wavenumbers are partitioned over S ranks of a
  // spectral group (pairs (m, T-m) dealt round-robin); this rank owns part
  // split_sp.  S = 1: unsplit (m_part = 0, m_k = m, Lp = L, lists null).
  int split_S, split_sp, Lp;
  int* m_part;      // [L] part owning m
  int* m_k;         // [L] position of m in its part's list
  int* own_m;       // [n_own_m] own wavenumbers, ascending (= k order)
  int n_own_m;
  int* own_work;    // analysis work items of own m
  int n_own_work;
  int* own_idx;     // own coefficient indices, ascending
  int n_own_idx;
  double2* fsyn_ext;  // part-major Fourier buffer [S][nb][J][Lp][4][2] (caller-owned)
  // H-free transforms (legendre_ponly.cu, table-streaming path): H = (1 - mu^2) dP/dmu
  // is replaced by the recurrence H_n = a_n P_{n-1} + b_n P_{n+1} (a_n = (n+1) eps_n,
  // b_n = -n eps_{n+1}, eps_n = sqrt((n^2 - m^2) / (4 n^2 - 1))), applied to the
  // coefficients: the synthesis runs 4 P transforms to degree T+1 and the analysis
  // 5 (A, B, C, D, E) whose neighbouring degrees the assembly combines; no H table
  int ponly;          // 1: active for unsplit plans (SDCSW_PONLY; default from T200)
  int rowsP, CP;      // P rows (degrees m..T+1, parity-sorted, padded to 8); extended triangle
  double* ptabP;      // [rowsP][J] (the analysis TMA map streams this)
  double* ptabP_s;    // [rowsP/4][J/8][8][4] synthesis fragment order
  int* rowoffP;       // [T+2]
  int* n_evenP;       // [T+1]
  int* rowP_n;        // [rowsP] degree k of each P row (-1: padding)
  int* moffP;         // [T+2] offsets of the extended triangle (T+2-m entries per m)
  int4* cvt_rows;     // [rowsP] xsyn rows of (m,k), (m,k-1), (m,k+1) (-1: none), P-triangle index
  double2* cvt_ab;    // [rowsP] (a_{k+1}, b_{k-1}): weights of X_{k+1}, X_{k-1}
  int4* prep_idx;     // [rowsP] coefficient indices of (m,k), (m,k-1), (m,k+1) (-1: none), m
  int4* coef_prow;    // [C] P row of (m,n), P row of (m,T+1) when n = T (else -1), n > m, n < T
  int2* asm_pos;      // [C] (extended-triangle index of (m,n), m)
  double2* asm_ab;    // [C] (a_n, b_n)
  int* anal_workP;    // [n_anal_workP] (m << 16 | 64-row block) over the P rows
  int n_anal_workP;
  int* own_workP;     // split plans: the work items of own m
  int n_own_workP;
  double* xsynP;      // [max_batch][rowsP][8] P-only synthesis operand (fragment order per batch)
  double* ghat;       // [max_batch][CP][10] P analyses of A, B, C, D, E to degree T+1
  alignas(64) unsigned long long tmapP[16];  // TMA map over ptabP
  alignas(64) unsigned long long gmapP[16];  // ring store map of the 5-slot analysis data
  int gmapP_rows;                             // rows per store box (0: plain stores)
  // planar problem (kind 1): N x N grid, spectra [N (kx)][NH = N/2 + 1 (ky)],
  // C = N * NH coefficients per field (lam = k^2 = laplacian symbol)
  int pn, pnh;
  double pf0, pnu;     // Coriolis parameter f0, hyperviscosity nu
  double* pkx;         // [N] x wavenumbers (2 pi fftfreq)
  double* pky;         // [NH] y wavenumbers (2 pi rfftfreq)
  double2* ptw;        // [N] exp(-2 pi i k / N)
  double2* pw1;        // [max_batch][4][N][NH] (U, V, zeta, Phi') after the column inverse FFTs
  double2* pw2;        // [max_batch][5][N][NH] row spectra of the five grid products
};
constexpr int kCoefCap = 4096;
constexpr int kEnsembleBatch = 16;  // plans for at least this many states per f_E are ensemble plans

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialization and waits for its predecessor's memory
// (griddepcontrol.wait) before reading anything the predecessor produced;
// constant plan data (tables, index lists, twiddles) is read before the wait.
// Dependents are released at exit, except by the ring kernel, which releases
// them before its output phase (measured).  The next kernel's launch and
// prologue then overlap the previous kernel's tail, in streams and graphs alike.
#ifdef __CUDACC__
// (Releasing dependents at kernel entry measured slower than the implicit
// release at exit, so SDCSW_PDL_ENTRY is empty unless SDCSW_EARLY_TRIGGER.)
#ifdef SDCSW_EARLY_TRIGGER
#define SDCSW_PDL_ENTRY() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#else
#define SDCSW_PDL_ENTRY()
#endif
#define SDCSW_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
// explicit release at a kernel-chosen point (per-kernel experiments: 0 = exit)
#define SDCSW_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#ifndef SDCSW_TRIG_RING
#define SDCSW_TRIG_RING 2  // measured: ring releases before its output phase
#endif
#ifndef SDCSW_TRIG_ANA
#define SDCSW_TRIG_ANA 0
#endif
#ifndef SDCSW_TRIG_SYN
#define SDCSW_TRIG_SYN 0
#endif
#endif
extern bool g_pdl;  // runtime switch (SDCSW_PDL=0 disables)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// error plumbing
void set_error(const std::string& msg);

// Device allocations of plans and steppers.  With SDCSW_GUARD=1 in the
// environment every allocation carries a 64 KiB canary in front and behind,
// checked when it is freed and by sdcsw_guard_check(): the in-library bounds
// check for out-of-range stores of the kernels (padding reads stay legal).
cudaError_t dev_alloc(void** p, size_t bytes);
cudaError_t dev_free(void* p);
template <typename T>
inline cudaError_t dev_alloc(T** p, size_t bytes) {
  return dev_alloc(reinterpret_cast<void**>(p), bytes);
}
int cuda_status(cudaError_t e, const char* where);

// Synthesis B operand ("xsyn"), 12 doubles per (packed table row r, batch
// entry b) in three parts of four:
//   part 0: U_P re, U_P im, V_P re, V_P im;  part 1: zeta re, zeta im, Phi re, Phi im;
//   part 2: U_H re, U_H im, V_H re, V_H im
// with U_P = i m chi / a, V_P = i m psi / a, U_H = -psi / a, V_H = chi / a.
// Fragment order for a batch of w entries: [row quad r/4][part][b][r % 4][4],
// so that the synthesis B fragment of a pair of entries (4 rows x 2 entries x
// 4 columns) is 32 consecutive doubles.  Element k of (r, b) is at
// xsyn_off(r, b, w) + (k / 4) * 16 w + k % 4; a row quad spans 12 w doubles per
// row, so rows [r0, r0 + 4q) are the contiguous range [12 w r0, 12 w (r0 + 4q)).
// Producers write only valid rows; padding rows of a buffer must stay zero.
constexpr int kXsyn = 12;

#ifdef __CUDACC__
__device__ __forceinline__ size_t xsyn_off(int r, int b, int w) {
  return ((size_t)(r >> 2) * 3 * w + b) * 16 + (r & 3) * 4;
}
// rec = xsyn_off(...) element pointer, pstride = 16 w (part stride)
__device__ __forceinline__ void write_xsyn_half(double* __restrict__ rec, size_t pstride, int ri,
                                                double phi, double zeta, double delta, double2 sc) {
  // ri = 0 holds real parts, ri = 1 imaginary parts; (x + i y)(-i s) = s y - i s x
  const double sm = sc.x, sa = sc.y;
  double* p1 = rec + pstride;
  double* p2 = rec + 2 * pstride;
  if (ri == 0) {
#if SDCSW_MUTATE_UCHI  // test-only mutation (node_math.cuh write_xsyn_full)
    rec[1] = sm * delta;
#else
    rec[1] = -sm * delta;  // U_P im
#endif
    rec[3] = -sm * zeta;   // V_P im
    p1[0] = zeta;
    p1[2] = phi;
    p2[0] = sa * zeta;     // U_H re
    p2[2] = -sa * delta;   // V_H re
  } else {
#if SDCSW_MUTATE_UCHI
    rec[0] = -sm * delta;
#else
    rec[0] = sm * delta;   // U_P re
#endif
    rec[2] = sm * zeta;    // V_P re
    p1[1] = zeta;
    p1[3] = phi;
    p2[1] = sa * zeta;     // U_H im
    p2[3] = -sa * delta;   // V_H im
  }
}

#endif

// P-only operand: 8 doubles per (P row, state) in two parts of four, part 0 =
// (U', V') (re, im) with U' = i m chi / a + sum of the recurrence terms of
// -psi / a, V' likewise of (i m psi / a, chi / a), part 1 = (zeta, Phi); same
// fragment order as xsyn with two parts: [row quad][part][b][r % 4][4].
constexpr int kXsynP = 8;
// P-only analysis data per (state, m, pair j): [j >> 2][fold S, A][j & 3][5 slots
// A, B, C, D (w_s-weighted), E (w_ke-weighted)][re, im] = 20 doubles per j
constexpr int kSlotsP = 5;
constexpr int kGhat = 2 * kSlotsP;  // doubles per (extended coefficient, state) of ghat
constexpr int kGanP = 4 * kSlotsP;  // doubles per (state, m, pair j) of the H-free analysis data
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int ganp_off(int j, int fold, int slot, int ri) {
  return ((j >> 2) * 2 + fold) * 40 + (j & 3) * 10 + slot * 2 + ri;
}

// the H-free transforms serve this plan's f_E (every launcher routes on it, split or not)
inline bool ponly_on(const Plan& p) { return p.kind == 0 && p.ponly && p.xsynP != nullptr; }

// Transform workspaces of one f_E chain (Fourier + analysis data); concurrent
// chains use disjoint batch slices of the plan's workspaces (the H-free path's
// analysis data is packed at 5 slots per (pair, m, fold) instead of 7).
struct Work {
  double2* fsyn;
  double2* gan;
  double* xsp;   // P-only operand slice (null unless ponly)
  double* ghat;  // P-only analysis output slice
};
inline Work plan_work(const Plan& p, int batch_offset = 0) {
  const size_t per = (size_t)p.J * p.L * 2;
  const bool po = ponly_on(p);
  Work w{p.fsyn + per * 4 * batch_offset, p.gan + per * (po ? kSlotsP : kNumSlots) * batch_offset,
         nullptr, nullptr};
  if (po) {
    w.xsp = p.xsynP + (size_t)batch_offset * p.rowsP * kXsynP;
    w.ghat = p.ghat + (size_t)batch_offset * p.CP * kGhat;
  }
  return w;
}

// launchers (return cudaError_t of the launch)
cudaError_t launch_synth_prep(const Plan& p, const double2* u, int nb, double* xsyn,
                              cudaStream_t s, int chunk = 0);
// split-mode synthesis into part split_sp of the external Fourier buffer
cudaError_t launch_synthesis_split(const Plan& p, const double* xsyn, int nb, cudaStream_t s);
// ring over all latitudes reading a part-major Fourier buffer (fsyn_ext)
cudaError_t launch_ring_split(const Plan& p, const Work& w, int nb, cudaStream_t s);
// split synthesis of own m published into every spectral peer's buffer, and
// the ring that waits for all parts (peer.cu)
struct SynDst;
struct RingPeer;
cudaError_t launch_synthesis_peer(const Plan& p, const double* xsyn, int nb, cudaStream_t s,
                                  const SynDst& d, int* step_counter);
cudaError_t launch_ring_peer(const Plan& p, const Work& w, const double2* fbase, int nb,
                             cudaStream_t s, const RingPeer& rp);
cudaError_t launch_synthesis(const Plan& p, const Work& w, const double* xsyn, int nb,
                             cudaStream_t s, int* step_counter);
cudaError_t launch_ring(const Plan& p, const Work& w, int nb, cudaStream_t s);
cudaError_t launch_analysis(const Plan& p, const Work& w, double2* fe, int nb, cudaStream_t s);
// ---------------------------------------------------------------------------
// Peer exchange of node-parallel dSDC (peer.cu).  Each rank owns one exchange
// buffer X = [2 parities][M nodes][2 (fe, fi)][3C] complex, mapped into every
// peer (CUDA IPC over NVLink), and a flag block.  Exchanges are numbered
// n = (epoch - 1) (K - 1) + k for full sweep k = 1..K-1 of the rank's epoch-th
// step (epoch: a device step counter, never reset), so every kernel derives n
// from device state and the captured graphs replay unchanged.
//   publish  the analysis (or a copy kernel) of sweep k stores the rank's
//            (fe, fi) into parity n & 1 of every rank's X (plain peer stores);
//   post     the next kernel that consumes exchange n (node kernel of sweep
//            k + 1, or the closing solve) first raises flag[rank] of every rank
//            to n - its own publishing grid has completed and flushed its
//            stores by then (griddepcontrol.wait); a system-scope fence
//            then orders the post (system-scope atomic max) after them;
//   wait     then spins until flag[q] >= n for all q (acquire) and reads
//            parity n & 1 locally.
// Two parities suffice: a rank publishes n + 2 only after passing the wait for
// n + 1, i.e. after every rank posted n + 1, which each rank does after its
// reads of exchange n have completed.
// ---------------------------------------------------------------------------
constexpr int kMaxPeers = 16;
struct PeerFlags {
  unsigned long long flag[kMaxPeers];  // flag[q]: last exchange rank q posted here
};
// Every device wait on a peer's post is bounded: after `limit_ns` (globaltimer)
// without the post, the waiter records (peer + 1, exchange number) in the
// exchange's error words and returns; later waits of the exchange see the
// error and do not wait again.  The host reports it as SDCSW_ERR_PEER (a peer
// that died or stopped stepping produces an error, not a hung GPU).
struct PeerTimeout {
  int* err;                      // [0] peer + 1 (0 = none), [1] channel, [2] exchange number
  unsigned long long limit_ns;
};
struct PeerWait {
  const PeerFlags* flags;   // local flag block (null: no exchange, plain pointers)
  const int* epoch;         // device step counter of the exchange (incremented per step)
  int k;                    // consumed exchange's sweep index within the step (1..K-1)
  int kx;                   // exchanges per step (K - 1)
  int world;
  long long par_stride;     // doubles between the two parities of X
  unsigned long long* post[kMaxPeers];  // &flags_q->flag[rank] of every rank q
  PeerTimeout to;
};
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// mbarrier / bulk-copy helpers (TMA engine; legendre_tma.cu, ring_fft.cu)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin (acquire, system scope) until *flag >= n; false after the time limit or
// if an earlier wait of this exchange already timed out (error recorded).
static __device__ __noinline__ bool wait_posted(const unsigned long long* flag, unsigned long long n,
                                         const PeerTimeout& to, int peer, int channel) {
  if (ld_acquire_sys(flag) >= n) return true;
  volatile int* err = to.err;
  if (err[0] != 0) return false;
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(flag) < n) {
    __nanosleep(64);
    if (global_ns() - t0 > to.limit_ns || err[0] != 0) {
      if (atomicCAS(to.err, 0, peer + 1) == 0) {
        err[1] = channel;
        err[2] = (int)n;
        __threadfence_system();
      }
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ unsigned long long exchange_number(const int* epoch, int k, int kx) {
  return (unsigned long long)(*epoch - 1) * (unsigned long long)kx + (unsigned long long)k;
}
// Post + wait; called by every thread of the CTA before any early return.
// Returns the parity offset (doubles) of exchange n in X.
__device__ __forceinline__ long long peer_wait(const PeerWait& pw) {
  if (pw.flags == nullptr) return 0;
  SDCSW_PDL_WAIT();  // the publishing grid (and the epoch increment) completed
  const unsigned long long n = exchange_number(pw.epoch, pw.k, pw.kx);
  if (threadIdx.x == 0) {
    // The data of exchange n were stored by this rank's previous grid, which
    // has completed (griddepcontrol.wait above).  Across devices the post is
    // ordered after those peer stores by a system-scope fence (its latency,
    // 4 us per exchange on B200, is the price of not relying on how NVLink
    // orders a later store against earlier striped ones); within one device
    // the kernel boundary already orders them.
    if (pw.world > 1) __threadfence_system();
    for (int q = 0; q < pw.world; ++q) atomicMax_system(pw.post[q], n);
    for (int q = 0; q < pw.world; ++q)
      if (!wait_posted(&pw.flags->flag[q], n, pw.to, q, 0)) break;
  }
  __syncthreads();
  return (long long)(n & 1) * pw.par_stride;
}
#endif

// Spectral split over peer memory (peer.cu): the S ranks of a spectral group
// exchange the synthesised Fourier coefficients of their wavenumbers once per
// f_E.  Fourier exchange n (n = fseq + 1, fseq counting this rank's completed
// exchanges) is written by every rank's synthesis into part sp of parity
// n & 1 of every spectral peer's part-major buffer; the ring kernel posts n
// into flag[sp] of every spectral peer, waits for all S posts, reads parity
// n & 1, and its last CTA to finish sets fseq = n (every CTA has read fseq by
// then).  Double buffering as for the node exchange.
struct SynDst {
  int n;                           // destinations (0: plain synthesis into fsyn)
  long long par_stride;            // double2 per parity of a Fourier exchange buffer
  const unsigned long long* fseq;  // completed Fourier exchanges of this rank
  double2* dst[kMaxPeers];         // part sp of every spectral peer's buffer (parity 0)
};
struct RingPeer {
  const PeerFlags* flags;          // local Fourier flag block (null: no exchange)
  unsigned long long* fseq;
  unsigned int* done;              // CTAs finished (reset by the last one)
  int world;
  long long par_stride;            // double2 per parity
  unsigned long long* post[kMaxPeers];  // &fourier flags of spectral peer q ->flag[sp]
  PeerTimeout to;
};

// Sweep-fused analysis (latency regime, one state, M <= kFuseMaxNodes): the
// epilogue takes f_E of every node straight from shared memory and runs the
// next sweep's node updates (mode 1) or the closing last-node solve (mode 2),
// so f_E never reaches HBM and the node kernels disappear from the step.
constexpr int kFuseMaxNodes = 6;
struct FuseArgs {
  int mode;                 // 1: next sweep's node updates; 2: closing solve; 3: serial SDC node;
                            // 4: publish f_E and f_I to the peers (node-parallel dSDC)
  int M, first;             // first: every node's tendencies are f_E(u0), f_I(u0)
  const double* u0;         // step-start state
  double* fi;               // f_I of the nodes [M][3C]: read, and (mode 1) updated in place
  double* u_out;            // mode 2: the step's result (may alias u0); mode 3: last node's
  double* xsyn;             // next synthesis operand (nb = M in mode 1, 1 in modes 2, 3)
  int* diverged;            // modes 2, 3: atomicMin(step index) on a non-finite result
  const int* step_counter;
  double phibar;
  // mode 3 (serial sweep, f_E of node m just computed; serial_update(m) and
  // serial_node(m + 1) of nodes.cu follow in the epilogue):
  double* fe_new;           // fe of node m (stored)
  const double* fe_old;     // fe of node m in the previous sweep (fe0 when first)
  const double* fi_old;     // fi of node m in the previous sweep (unused when first)
  const double* fi_new;     // fi of node m of this sweep
  double* corr;             // running correction, updated in place
  const double* quad_next;  // quad of node m + 1 (null: m is the sweep's last node)
  const double* fi_old_next;  // fi of node m + 1 in the previous sweep (unused when first)
  double* fi_new_next;      // fi of node m + 1 (out)
  int use_corr;             // m > 0: the correction exists
  // mode 4 (node-parallel publish, peer.cu): f_E of this rank's nodes
  // [peer_lo, peer_lo + nb) and their f_I (peer_fi, [nb][3C]) are stored into
  // parity n & 1 of every rank's exchange buffer
  int peer_world, peer_lo, peer_k, peer_kx;  // exchange n = (epoch - 1) kx + k
  const int* peer_epoch;
  const double* peer_fi;
  double* peer_x[kMaxPeers];
  double cf[kFuseMaxNodes * (kFuseMaxNodes + 4)];  // mode 1: [M][M+4]; mode 2: [M+4];
                                                   // mode 3: we, wi, alpha, a_phi, a2_phi
};
// the TMA analysis (and the fragment-order analysis data it reads) is in use
inline bool tma_active(const Plan& p) { return p.tma_ok && p.anal_wj == 4; }
inline bool fuse_supported(const Plan& p, int M) {
  return p.kind == 0 && !p.tma_ok && p.own_idx == nullptr && M >= 1 && M <= kFuseMaxNodes;
}
cudaError_t launch_analysis_fused(const Plan& p, const Work& w, int nb, const FuseArgs& fz,
                                  cudaStream_t s);
cudaError_t launch_f_impl(const Plan& p, const double2* u, double2* fi, int nb, cudaStream_t s);
// coefficient pointers below are HOST memory; values travel as kernel parameters
// opt-in collocation-residual norms of the sweep kernel (nodes.cu resid_block)
struct ResidArgs {
  const double* u_prev;  // previous iterate's node values [count][3C] complex
  double* part;          // per-block partials [count * 3][blocks]
  unsigned* count;       // blocks finished (0 between calls)
  double* out;           // [count][3] norms (device)
};
cudaError_t launch_solve(const Plan& p, const double* coef_host, const double2* beta, double2* u,
                         int nb, cudaStream_t s);
cudaError_t launch_sweep_nodes(const Plan& p, int M, int node_lo, int count, const double* coef_host,
                               const double2* u0, const double2* fe, long long fe_stride,
                               const double2* fi, long long fi_stride, int first, double2* u_out,
                               double2* fi_out, double* xsyn_out, cudaStream_t s, int members = 1,
                               long long fe_mstride = 0, long long fi_mstride = 0, int chunk = 0,
                               const PeerWait* pw = nullptr, const ResidArgs* ra = nullptr);
cudaError_t launch_final_node(const Plan& p, int M, const double* coef_host, const double2* u0,
                              const double2* fe, long long fe_stride, const double2* fi,
                              long long fi_stride, int first, double2* u_out, int* diverged,
                              const int* step_counter, double* xsyn_out, cudaStream_t s,
                              int members = 1, long long fe_mstride = 0, long long fi_mstride = 0,
                              const PeerWait* pw = nullptr);
cudaError_t launch_serial_quad(const Plan& p, int M, const double* w_host, const double2* u0,
                               const double2* fe, long long fe_stride, const double2* fi,
                               long long fi_stride, int first, double2* quad, cudaStream_t s);
cudaError_t launch_serial_node(const Plan& p, int M, int m, const double* coef_host,
                               const double2* quad, const double2* corr, const double2* u0,
                               const double2* fi_old, int first, double2* u_out, double2* u_out2,
                               double2* fi_new, int* diverged, const int* step_counter,
                               double* xsyn_out, cudaStream_t s);
cudaError_t launch_serial_update(const Plan& p, int m, double we, double wi, double2* corr,
                                 const double2* fe_new, const double2* fe_old,
                                 const double2* fi_new, const double2* fi_old, const double2* u0,
                                 int first, cudaStream_t s);
cudaError_t launch_check_finite(const double* x, long long n, int* flag, cudaStream_t s);
cudaError_t launch_axpy(long long n, const double* x, double w, const double* y, double* out,
                        cudaStream_t s);

cudaError_t make_table_maps(Plan& p);
// H-free path (legendre_ponly.cu): plan tables / maps, and the f_E chain stages
cudaError_t ponly_setup(Plan& p, const double* ptab, const int* rowoff, const int* row_n,
                        const double* mu_north);
void ponly_free(Plan& p);
// (the generic launchers below route to these when ponly_on(p); split plans pass
// their own wavenumbers / work items)
cudaError_t launch_synthesis_ponly(const Plan& p, double2* fsyn, const int* mlist, int nm, int Lp,
                                   double* xsp, const double* xsyn, int nb, cudaStream_t s,
                                   int* step_counter, const SynDst& sd);
cudaError_t launch_analysis_ponly(const Plan& p, const Work& w, double2* fe, int nb, cudaStream_t s);
// H-free f_E straight from nb states u (the P-only operand built from the states, no
// 12-double records): the dSDC stepper's path on H-free plans
cudaError_t f_expl_states_ponly(const Plan& p, const Work& w, const double2* u, double2* fe, int nb,
                                cudaStream_t s, int* step_counter);
// H-free f_E from the P-only operand xsp a node kernel already wrote (padding rows zero)
cudaError_t f_expl_operand_ponly(const Plan& p, const Work& w, const double* xsp, double2* fe, int nb,
                                 cudaStream_t s);
// the dSDC sweep's node updates writing f_I and the P-only synthesis operand of the new node
// states (nodes.cu k_sweep_nodes_po; no node states stored, no operand kernel)
cudaError_t launch_sweep_nodes_po(const Plan& p, int M, int node_lo, int count, const double* coef_host,
                                  const double2* u0, const double2* fe, long long fe_stride,
                                  const double2* fi, long long fi_stride, int first, double2* fi_out,
                                  double* xsp, cudaStream_t s, int members, long long fe_mstride,
                                  long long fi_mstride);
cudaError_t make_gan_maps(Plan& p);
cudaError_t configure_synthesis_bulk();
cudaError_t configure_analysis_bulk();
bool synthesis_bulk_ok(const Plan& p, int nb);
cudaError_t launch_synthesis_bulk(const Plan& p, double2* fsyn, const int* mlist, int nm, int Lp,
                                  const double* xsyn, int nb, cudaStream_t s, int* step_counter,
                                  const SynDst& sd);
cudaError_t configure_synthesis();
bool launch_analysis_tma(const Plan& p, const Work& w, double2* fe, int nb, cudaStream_t s,
                         cudaError_t* err);

// planar f_E: column inverse FFTs -> row FFTs with the grid products -> column
// forward FFTs and the tendency assembly (planar.cu)
cudaError_t planar_f_expl(const Plan& p, const double2* u, double2* fe, int nb, cudaStream_t s,
                          int* step_counter);
bool planar_supported(int n);
cudaError_t configure_planar(int n);

// f_E = (prep) -> synthesis -> ring -> analysis; f_expl_prepped starts from an
// xsyn operand a producer kernel already wrote
cudaError_t f_expl(Plan& p, const double2* u, double2* fe, int nb, cudaStream_t s,
                   int* step_counter);
cudaError_t f_expl_prepped(const Plan& p, const Work& w, const double* xsyn, double2* fe, int nb,
                           cudaStream_t s, int* step_counter, int chunk = 0);

}  // namespace sdcsw

// the C-ABI plan handle (include/sdcsw.h)
struct sdcsw_plan {
  sdcsw::Plan p;
  bool alive;
};

