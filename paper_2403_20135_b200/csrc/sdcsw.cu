// C ABI of libsdcsw.so (declared in include/sdcsw.h): plan lifecycle, the
// problem operations, the fused sweep operations and the device-resident
// stepper that replays one captured CUDA graph per time step.
#include <climits>
#include <cstdlib>
#include <cmath>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "internal.cuh"

namespace sdcsw {

static thread_local std::string g_error;

static bool pdl_default() {
  const char* e = getenv("SDCSW_PDL");
  return !(e && e[0] == '0');
}
bool g_pdl = pdl_default();

void set_error(const std::string& msg) { g_error = msg; }

// ---- guarded allocations (SDCSW_GUARD=1) ----------------------------------------
namespace {
constexpr size_t kGuardBytes = 64 << 10;
constexpr unsigned char kGuardFill = 0xA5;
struct GuardRec {
  char* base;
  size_t bytes;
};
std::mutex g_guard_mu;
std::vector<GuardRec> g_guards;
long long g_guard_bad = 0;  // corrupted canary bytes of allocations already freed

bool guard_on() {
  static const bool on = [] {
    const char* e = std::getenv("SDCSW_GUARD");
    return e != nullptr && e[0] == '1';
  }();
  return on;
}

long long guard_scan(const GuardRec& r) {
  std::vector<unsigned char> h(2 * kGuardBytes);
  if (cudaMemcpy(h.data(), r.base, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(h.data() + kGuardBytes, r.base + kGuardBytes + r.bytes, kGuardBytes,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return 2 * (long long)kGuardBytes;
  long long bad = 0;
  for (unsigned char c : h) bad += c != kGuardFill;
  return bad;
}
}  // namespace

cudaError_t dev_alloc(void** p, size_t bytes) {
  if (!guard_on()) return cudaMalloc(p, bytes);
  char* base = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuardBytes);
  if (e != cudaSuccess) return e;
  e = cudaMemset(base, kGuardFill, kGuardBytes);
  if (e == cudaSuccess) e = cudaMemset(base + kGuardBytes + bytes, kGuardFill, kGuardBytes);
  if (e != cudaSuccess) {
    cudaFree(base);
    return e;
  }
  std::lock_guard<std::mutex> lock(g_guard_mu);
  g_guards.push_back({base, bytes});
  *p = base + kGuardBytes;
  return cudaSuccess;
}

cudaError_t dev_free(void* p) {
  if (!guard_on() || p == nullptr) return cudaFree(p);
  std::lock_guard<std::mutex> lock(g_guard_mu);
  for (size_t i = 0; i < g_guards.size(); ++i) {
    if (g_guards[i].base + kGuardBytes != p) continue;
    cudaDeviceSynchronize();
    g_guard_bad += guard_scan(g_guards[i]);
    char* base = g_guards[i].base;
    g_guards.erase(g_guards.begin() + i);
    return cudaFree(base);
  }
  return cudaFree(p);
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return SDCSW_OK;
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return SDCSW_ERR_CUDA;
}

cudaError_t configure_ring(size_t smem);
size_t ring_smem_bytes(int nlon);
bool ring_pass_twiddles(int nlon, const double2* w, std::vector<double2>& out);

bool ring_supported(int nlon);

cudaError_t f_expl_prepped(const Plan& p, const Work& w, const double* xsyn, double2* fe, int nb,
                           cudaStream_t s, int* step_counter, int chunk) {
  // chunk > 0: the operand is chunk-major ([nb/chunk][rows][chunk][kXsyn]) and
  // each chunk runs synthesis -> ring -> analysis on its own (L2-resident)
  const int ch = chunk > 0 && chunk < nb ? chunk : nb;
  for (int b0 = 0; b0 < nb; b0 += ch) {
    const int n = nb - b0 < ch ? nb - b0 : ch;
    const double* xs = xsyn + (size_t)b0 * p.rows * kXsyn;
    double2* out = fe + (size_t)b0 * 3 * p.C;
    cudaError_t e = launch_synthesis(p, w, xs, n, s, b0 == 0 ? step_counter : nullptr);
    if (e != cudaSuccess) return e;
    e = launch_ring(p, w, n, s);
    if (e != cudaSuccess) return e;
    e = launch_analysis(p, w, out, n, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t f_expl(Plan& p, const double2* u, double2* fe, int nb, cudaStream_t s,
                   int* step_counter) {
  cudaError_t e;
  if (p.xsyn_nb != nb) {  // record layout changes: padding rows must read as zero
    e = cudaMemsetAsync(p.xsyn, 0, (size_t)p.rows * nb * kXsyn * sizeof(double), s);
    if (e != cudaSuccess) return e;
    p.xsyn_nb = nb;
  }
  e = launch_synth_prep(p, u, nb, p.xsyn, s);
  if (e != cudaSuccess) return e;
  return f_expl_prepped(p, plan_work(p), p.xsyn, fe, nb, s, step_counter);
}

template <typename T>
static cudaError_t upload(T** dst, const T* src, size_t n, size_t pad = 0) {
  cudaError_t e = dev_alloc(dst, (n + pad) * sizeof(T));
  if (e != cudaSuccess) return e;
  if (pad) cudaMemset(*dst + n, 0, pad * sizeof(T));
  if (n) e = cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace sdcsw

using namespace sdcsw;

struct sdcsw_stepper {
  sdcsw_plan* plan;
  int mode, M, K;
  std::vector<double> coef;
  double2* buf;  // all sweep storage in one allocation
  size_t S;      // one state, in double2
  double2 *fe0, *fe, *fi, *ustage, *quad, *corr, *feB, *fiB;
  double *xsyn1, *xsynM;  // synthesis operands (nb = 1 / node groups); padding rows stay zero
  int chains;             // concurrent node chains per sweep (graph branches)
  int members;            // ensemble members advanced together (batched GEMM columns)
  int sequential;         // 1: node updates one after another (DIAGONAL_SEQUENTIAL analogue)
  int fuse;               // 1: node updates run in the analysis epilogue (launch_analysis_fused)
  int ncreated;           // side streams created
  cudaEvent_t prof[40];   // stage events of a profiled step (created on demand)
  bool prof_ready;
  cudaStream_t side[16];
  cudaEvent_t ev_fork, ev_join[16];
  int* flags;    // [0] first diverged step (INT_MAX = none), [1] step counter
  cudaStream_t cap;
  cudaGraph_t graph;
  cudaGraphExec_t exec;     // one step
  cudaGraph_t graphK;
  cudaGraphExec_t execK;    // graph_steps steps back to back (PDL across step boundaries)
  int graph_steps;
  double* graph_u;
  int launches;
  size_t nstates;  // state-sized buffers in buf
  int sprep;       // H-free dSDC: f_E builds its P-only operand from the node states (ustage)
  int nodes_po;    // H-free dSDC: the sweep's node kernel writes the P-only operand itself
  sdcsw_sweep_hook hook;  // per-sweep host callback of sdcsw_stepper_step_hooked (else null)
  void* hook_user;
};

extern "C" {

const char* sdcsw_last_error(void) { return g_error.c_str(); }
int sdcsw_version(void) { return 1; }

int sdcsw_guard_check(long long* corrupted_bytes, int* live_allocations) {
  if (!corrupted_bytes || !live_allocations) {
    set_error("sdcsw_guard_check: null argument");
    return SDCSW_ERR_PARAM;
  }
  if (!guard_on()) {
    *corrupted_bytes = 0;
    *live_allocations = -1;
    return SDCSW_OK;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_status(e, "sdcsw_guard_check");
  std::lock_guard<std::mutex> lock(g_guard_mu);
  long long bad = g_guard_bad;
  for (const GuardRec& r : g_guards) bad += guard_scan(r);
  *corrupted_bytes = bad;
  *live_allocations = (int)g_guards.size();
  return SDCSW_OK;
}

int sdcsw_guard_selftest(void) {
  unsigned char* q = nullptr;
  cudaError_t e = dev_alloc(&q, 256);
  if (e == cudaSuccess) e = cudaMemset(q + 255, 0, 2);  // the second byte is out of bounds
  if (e == cudaSuccess) e = dev_free(q);
  return cuda_status(e, "sdcsw_guard_selftest");
}

int sdcsw_plan_create(int device, const sdcsw_config* cfg, const double* mu_north,
                      const double* w_north, const double* ptab, const double* htab,
                      const int* rowoff, const int* n_even, const int* row_n, const double* lam,
                      sdcsw_plan** out) {
  if (!cfg || !out || !mu_north || !w_north || !ptab || !htab || !rowoff || !n_even || !row_n ||
      !lam) {
    set_error("sdcsw_plan_create: null argument");
    return SDCSW_ERR_PARAM;
  }
  const int T = cfg->trunc, nlat = cfg->nlat, nlon = cfg->nlon;
  if (T < 1 || nlat % 2 || nlat < T + 1 || (nlat / 2) % 16 || nlon < 2 * T + 2 || nlon > 1536 ||
      cfg->max_batch < 1 || T > 4000) {
    set_error("sdcsw_plan_create: unsupported size (need nlat/2 % 16 == 0, 2T+2 <= nlon <= 1536)");
    return SDCSW_ERR_PARAM;
  }
  if (!ring_supported(nlon)) {
    set_error("sdcsw_plan_create: nlon must be one of 96, 192, 384, 768, 1536 (3*2^k)");
    return SDCSW_ERR_PARAM;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  sdcsw_plan* h = new (std::nothrow) sdcsw_plan();
  if (!h) {
    set_error("out of host memory");
    return SDCSW_ERR_PARAM;
  }
  std::memset(&h->p, 0, sizeof(Plan));
  Plan& p = h->p;
  p.device = device;
  p.T = T; p.nlat = nlat; p.nlon = nlon; p.J = nlat / 2; p.L = T + 1;
  p.C = (T + 1) * (T + 2) / 2;
  p.max_batch = cfg->max_batch;
  p.radius = cfg->radius; p.omega = cfg->omega; p.phibar = cfg->phibar;
  p.rows = rowoff[T + 1];
  const int J = p.J, C = p.C;

  std::vector<int> moff(T + 2);
  for (int m = 0; m <= T + 1; ++m) moff[m] = m * (T + 1) - m * (m - 1) / 2;
  std::vector<double> inv_nn(C), wsyn(J), wke(J);
  std::vector<double2> xscale(C);
  std::vector<int> idx_row(C, -1);
  for (int m = 0; m <= T; ++m)
    for (int n = m; n <= T; ++n) {
      const int idx = moff[m] + n - m;
      inv_nn[idx] = n == 0 ? 0.0 : 1.0 / (double(n) * (n + 1.0));
      xscale[idx] = make_double2((double)m * cfg->radius * inv_nn[idx], cfg->radius * inv_nn[idx]);
    }
  for (int m = 0; m <= T; ++m)
    for (int r = rowoff[m]; r < rowoff[m + 1]; ++r)
      if (row_n[r] >= 0) idx_row[moff[m] + row_n[r] - m] = r;
  for (int i = 0; i < C; ++i)
    if (idx_row[i] < 0) {
      set_error("sdcsw_plan_create: row_n does not cover every coefficient");
      delete h;
      return SDCSW_ERR_PARAM;
    }
  const double twopi = 6.283185307179586476925286766559;
  for (int j = 0; j < J; ++j) {
    const double mu = mu_north[j];
    wsyn[j] = twopi * w_north[j] / (p.radius * ((1.0 - mu) * (1.0 + mu)));
    wke[j] = twopi * w_north[j];
  }
  std::vector<double2> tw(nlon);
  for (int i = 0; i < nlon; ++i) {
    const long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)i / nlon;
    tw[i] = make_double2((double)cosl(a), (double)sinl(a));
  }
  // FFT radices: 4s, then a 2 if needed, then the 3
  FftPlan fp;
  std::memset(&fp, 0, sizeof(fp));
  fp.n = nlon;
  int rem = nlon, ns = 0, k2 = 0;
  bool three = rem % 3 == 0;
  if (three) rem /= 3;
  while (rem > 1) { rem /= 2; ++k2; }
  // 2^k2 = 8^a 4^b (2 if k2 == 1): fewest passes
  int n8 = k2 / 3, n4 = 0, n2 = 0;
  if (k2 % 3 == 1) { if (n8 > 0) { n8 -= 1; n4 = 2; } else { n2 = 1; } }
  if (n2) {
    set_error("sdcsw_plan_create: nlon too small (radix-2 pass not supported)");
    delete h;
    return SDCSW_ERR_PARAM;
  }
  if (k2 % 3 == 2) n4 = 1;
  for (int q = 0; q < n8; ++q) fp.radix[ns++] = 8;
  for (int q = 0; q < n4; ++q) fp.radix[ns++] = 4;
  for (int q = 0; q < n2; ++q) fp.radix[ns++] = 2;
  if (three) fp.radix[ns++] = 3;
  fp.nstages = ns;
  p.fft = fp;
  // analysis work list
  std::vector<int> work;
  // row tiles per CTA: small truncations split K over the 4 warps (more warps
  // in flight), large ones give each warp its own row tile (B reuse via L1)
  // (from T200 the table-streaming analysis runs, which takes 4 row tiles per CTA)
  // ensemble plans (batches of at least kEnsembleBatch states) take the
  // table-streaming analysis at any truncation: 64-member T127 ensemble
  // analysis 504 -> 297 us per 256-state launch, c4 13.3k -> 15.3k member-steps/s
  p.ensemble = p.max_batch >= kEnsembleBatch;
  p.anal_wj = T < 200 && !p.ensemble ? 1 : 4;
  p.synth_wj = T < 200 ? 1 : (T < 400 ? 2 : 4);
  // cp.async-pipelined synthesis: -1 = automatic (see synthesis_impl)
  p.syn_cp = -1;
  if (const char* env = getenv("SDCSW_SYN_CP")) p.syn_cp = atoi(env);
  p.ana_nb = 0;
  if (const char* env = getenv("SDCSW_ANA_NB")) p.ana_nb = atoi(env);
  p.ana_bulk = 1;
  if (const char* env = getenv("SDCSW_ANA_BULK")) p.ana_bulk = atoi(env);
  p.syn_bulk = -1;
  if (const char* env = getenv("SDCSW_SYN_BULK")) p.syn_bulk = atoi(env);
  if (const char* env = getenv("SDCSW_ANAL_WJ")) p.anal_wj = atoi(env);
  if (const char* env = getenv("SDCSW_SYNTH_WJ")) p.synth_wj = atoi(env);
  while ((J / kRowsPerWarp) % p.synth_wj) p.synth_wj /= 2;
  for (int m = 0; m <= T; ++m) {
    const int rows = rowoff[m + 1] - rowoff[m];
    const int per = kRowsPerWarp * p.anal_wj;
    for (int rb = 0; rb * per < rows; ++rb) work.push_back((m << 16) | rb);
  }
  p.n_anal_work = (int)work.size();
  std::vector<int> work4;
  for (int m = 0; m <= T; ++m) {
    const int rows = rowoff[m + 1] - rowoff[m];
    for (int rb = 0; rb * 4 * kRowsPerWarp < rows; ++rb) work4.push_back((m << 16) | rb);
  }
  p.n_anal_work4 = (int)work4.size();
  p.ring_threads = 256;
  p.ring_smem = ring_smem_bytes(nlon);
  std::vector<double2> twp;
  ring_pass_twiddles(nlon, tw.data(), twp);

  const size_t tab = (size_t)p.rows * J;
  // fragment-order copies (coalesced 256-byte A-fragment loads in both GEMMs)
  std::vector<double> pa(tab), ha(tab), ps(tab), hs(tab);
  for (int r = 0; r < p.rows; ++r)
    for (int j = 0; j < J; ++j) {
      const size_t src = (size_t)r * J + j;
      const size_t a = (((size_t)(r / 8) * (J / 4) + j / 4) * 8 + r % 8) * 4 + j % 4;
      const size_t q = (((size_t)(r / 4) * (J / 8) + j / 8) * 8 + j % 8) * 4 + r % 4;
      pa[a] = ptab[src];
      ha[a] = htab[src];
      ps[q] = ptab[src];
      hs[q] = htab[src];
    }
  if ((e = upload(&p.ptab, ptab, tab, (size_t)16 * J)) != cudaSuccess ||
      (e = upload(&p.htab, htab, tab, (size_t)16 * J)) != cudaSuccess ||
      (e = upload(&p.ptab_a, pa.data(), tab, (size_t)16 * J)) != cudaSuccess ||
      (e = upload(&p.htab_a, ha.data(), tab, (size_t)16 * J)) != cudaSuccess ||
      (e = upload(&p.ptab_s, ps.data(), tab, (size_t)16 * J)) != cudaSuccess ||
      (e = upload(&p.htab_s, hs.data(), tab, (size_t)16 * J)) != cudaSuccess ||
      (e = upload(&p.rowoff, rowoff, (size_t)T + 2)) != cudaSuccess ||
      (e = upload(&p.n_even, n_even, (size_t)T + 1)) != cudaSuccess ||
      (e = upload(&p.row_n, row_n, (size_t)p.rows, 16)) != cudaSuccess ||
      (e = upload(&p.moff, moff.data(), moff.size())) != cudaSuccess ||
      (e = upload(&p.lam, lam, (size_t)C)) != cudaSuccess ||
      (e = upload(&p.inv_nn, inv_nn.data(), inv_nn.size())) != cudaSuccess ||
      (e = upload(&p.xscale, xscale.data(), xscale.size())) != cudaSuccess ||
      (e = upload(&p.idx_row, idx_row.data(), idx_row.size())) != cudaSuccess ||
      (e = dev_alloc(&p.xsyn, (size_t)p.rows * p.max_batch * kXsyn * sizeof(double))) != cudaSuccess ||
      (e = upload(&p.mu, mu_north, (size_t)J)) != cudaSuccess ||
      (e = upload(&p.wsyn, wsyn.data(), wsyn.size())) != cudaSuccess ||
      (e = upload(&p.wke, wke.data(), wke.size())) != cudaSuccess ||
      (e = upload(&p.twiddle, twp.data(), twp.size())) != cudaSuccess ||
      (e = upload(&p.anal_work, work.data(), work.size())) != cudaSuccess ||
      (e = upload(&p.anal_work4, work4.data(), work4.size())) != cudaSuccess ||
      (e = dev_alloc(&p.fsyn, (size_t)p.max_batch * J * p.L * 8 * sizeof(double2))) != cudaSuccess ||
      (e = dev_alloc(&p.gan, (size_t)p.max_batch * J * p.L * kNumSlots * 2 * sizeof(double2))) !=
          cudaSuccess ||
      (e = dev_alloc(&p.coef_dev, kCoefCap * sizeof(double))) != cudaSuccess ||
      // residual sweeps: [6 nodes x 3 fields][blocks] partials + last-block counter,
      // allocated here so the opt-in call never allocates (or is half-built) under capture
      (e = dev_alloc(&p.resid_part, 18 * (size_t)((C + 255) / 256) * sizeof(double))) != cudaSuccess ||
      (e = dev_alloc(&p.resid_count, sizeof(unsigned))) != cudaSuccess ||
      (e = cudaMemset(p.resid_count, 0, sizeof(unsigned))) != cudaSuccess ||
      (e = configure_ring(p.ring_smem)) != cudaSuccess ||
      (e = configure_synthesis()) != cudaSuccess ||
      (e = configure_synthesis_bulk()) != cudaSuccess ||
      (e = configure_analysis_bulk()) != cudaSuccess ||
      (e = make_table_maps(p)) != cudaSuccess ||
      (e = make_gan_maps(p)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess) {
    int st = cuda_status(e, "sdcsw_plan_create");
    void* ptrs[] = {p.ptab, p.htab, p.rowoff, p.n_even, p.row_n, p.moff, p.lam, p.inv_nn, p.mu,
                    p.wsyn, p.wke, p.twiddle, p.anal_work, p.fsyn, p.gan, p.coef_dev,
                    p.xscale, p.idx_row, p.xsyn, p.anal_work4, p.ptab_a, p.htab_a,
                    p.ptab_s, p.htab_s, p.resid_part, p.resid_count};
    for (void* q : ptrs)
      if (q) dev_free(q);
    delete h;
    return st;
  }
  p.xsyn_nb = -1;
  p.split_S = 1;
  p.split_sp = 0;
  p.Lp = p.L;
  {
    // Chunk big f_E batches so that one chunk's Fourier + analysis workspaces
    // (22 complex per (pair, m) and state) and the tables fit in ~half the L2;
    // only when the tables themselves are L2-resident (otherwise batching
    // amortises their HBM stream instead).  SDCSW_FE_CHUNK overrides.
    const double per_state = (double)J * p.L * 22 * sizeof(double2);
    const double tables = 2.0 * p.rows * J * sizeof(double);
    // measured on B200: chunking the c4 ensemble (T127, 256 states) to keep
    // the workspaces L2-resident was slower than one big batch, so it is off
    // unless requested
    (void)per_state;
    (void)tables;
    p.fe_chunk = 0;
    if (const char* env = getenv("SDCSW_FE_CHUNK")) p.fe_chunk = atoi(env);
  }
  // H-free transforms (legendre_ponly.cu) for the table-streaming path (T >= 200 and
  // ensemble plans); SDCSW_PONLY = 0 / 1 overrides the default
  {
    int po = 1;
    if (const char* env = getenv("SDCSW_PONLY")) po = atoi(env);
    if (po && tma_active(p)) {
      if (ponly_setup(p, ptab, rowoff, row_n, mu_north) == cudaSuccess) {
        p.ponly = 1;
      } else {
        cudaGetLastError();  // not built: the P/H path serves the plan
        p.ponly = 0;
      }
    }
  }
  h->alive = true;
  *out = h;
  return SDCSW_OK;
}

int sdcsw_plan_destroy(sdcsw_plan* h) {
  if (!h || !h->alive) {
    set_error("sdcsw_plan_destroy: invalid handle");
    return SDCSW_ERR_STATE;
  }
  cudaSetDevice(h->p.device);
  cudaDeviceSynchronize();
  Plan& p = h->p;
  ponly_free(p);
  for (void* q : {(void*)p.m_part, (void*)p.m_k, (void*)p.own_m, (void*)p.own_work, (void*)p.own_idx,
                  (void*)p.own_workP})
    if (q) dev_free(q);
  void* ptrs[] = {p.ptab, p.htab, p.rowoff, p.n_even, p.row_n, p.moff, p.lam, p.inv_nn, p.mu,
                  p.wsyn, p.wke, p.twiddle, p.anal_work, p.fsyn, p.gan, p.coef_dev,
                  p.xscale, p.idx_row, p.xsyn, p.anal_work4, p.pkx, p.pky, p.ptw, p.pw1, p.pw2,
                  p.ptab_a, p.htab_a, p.ptab_s, p.htab_s, p.resid_part, p.resid_count};
  for (void* q : ptrs)
    if (q) dev_free(q);
  h->alive = false;
  delete h;
  return SDCSW_OK;
}

int sdcsw_plan_create_planar(int device, const sdcsw_planar_config* cfg, const double* kx,
                             const double* ky, const double* lam, sdcsw_plan** out) {
  if (!cfg || !out || !kx || !ky || !lam) {
    set_error("sdcsw_plan_create_planar: null argument");
    return SDCSW_ERR_PARAM;
  }
  const int n = cfg->n_grid;
  if (!planar_supported(n) || cfg->max_batch < 1 || !(cfg->mean_geopotential > 0.0) ||
      cfg->hyperviscosity < 0.0) {
    set_error("sdcsw_plan_create_planar: n_grid must be 8, 12, 16, 24, ..., 768 or 1024 "
              "(2^k or 3*2^k), max_batch >= 1, mean_geopotential > 0, hyperviscosity >= 0");
    return SDCSW_ERR_PARAM;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  sdcsw_plan* h = new (std::nothrow) sdcsw_plan();
  if (!h) {
    set_error("out of host memory");
    return SDCSW_ERR_PARAM;
  }
  std::memset(&h->p, 0, sizeof(Plan));
  Plan& p = h->p;
  p.kind = 1;
  p.device = device;
  p.pn = n;
  p.pnh = n / 2 + 1;
  p.C = n * p.pnh;
  p.max_batch = cfg->max_batch;
  p.phibar = cfg->mean_geopotential;
  p.pf0 = cfg->coriolis;
  p.pnu = cfg->hyperviscosity;
  p.split_S = 1;
  p.xsyn_nb = -1;
  std::vector<double2> tw(n);
  for (int k = 0; k < n; ++k) {
    const long double a = -2.0L * 3.14159265358979323846264338327950288L * k / n;
    tw[k] = make_double2((double)cosl(a), (double)sinl(a));
  }
  const size_t wbytes = (size_t)p.max_batch * p.C * sizeof(double2);
  if ((e = upload(&p.pkx, kx, (size_t)n)) != cudaSuccess ||
      (e = upload(&p.pky, ky, (size_t)p.pnh)) != cudaSuccess ||
      (e = upload(&p.lam, lam, (size_t)p.C)) != cudaSuccess ||
      (e = upload(&p.ptw, tw.data(), tw.size())) != cudaSuccess ||
      (e = dev_alloc(&p.pw1, 4 * wbytes)) != cudaSuccess ||
      (e = dev_alloc(&p.pw2, 5 * wbytes)) != cudaSuccess ||
      (e = dev_alloc(&p.coef_dev, kCoefCap * sizeof(double))) != cudaSuccess ||
      (e = configure_planar(n)) != cudaSuccess) {
    const int st = cuda_status(e, "sdcsw_plan_create_planar");
    for (void* q : {(void*)p.pkx, (void*)p.pky, (void*)p.lam, (void*)p.ptw, (void*)p.pw1,
                    (void*)p.pw2, (void*)p.coef_dev})
      if (q) dev_free(q);
    delete h;
    return st;
  }
  h->alive = true;
  *out = h;
  return SDCSW_OK;
}

static int check_spherical(sdcsw_plan* h, const char* where) {
  if (h->p.kind != 0) {
    set_error(std::string(where) + ": spherical plans only");
    return SDCSW_ERR_STATE;
  }
  return SDCSW_OK;
}

static int check_plan(sdcsw_plan* h, int nb, const char* where) {
  if (!h || !h->alive) {
    set_error(std::string(where) + ": invalid plan handle");
    return SDCSW_ERR_STATE;
  }
  if (nb < 0 || nb > h->p.max_batch) {
    set_error(std::string(where) + ": batch exceeds plan max_batch");
    return SDCSW_ERR_PARAM;
  }
  return SDCSW_OK;
}

int sdcsw_f_expl(sdcsw_plan* h, const double* u, double* fe, int nb, void* stream) {
  int st = check_plan(h, nb, "sdcsw_f_expl");
  if (st) return st;
  if (h->p.split_S > 1) {
    set_error("sdcsw_f_expl: plan is spectrally split; use sdcsw_split_f_expl_begin/end");
    return SDCSW_ERR_STATE;
  }
  if (nb == 0) return SDCSW_OK;
  if (h->p.kind == 1)
    return cuda_status(planar_f_expl(h->p, (const double2*)u, (double2*)fe, nb,
                                     (cudaStream_t)stream, nullptr),
                       "sdcsw_f_expl");
  return cuda_status(f_expl(h->p, (const double2*)u, (double2*)fe, nb, (cudaStream_t)stream, nullptr),
                     "sdcsw_f_expl");
}

int sdcsw_f_impl(sdcsw_plan* h, const double* u, double* fi, int nb, void* stream) {
  int st = check_plan(h, 1, "sdcsw_f_impl");
  if (st) return st;
  if (nb < 0) return SDCSW_ERR_PARAM;
  if (nb == 0) return SDCSW_OK;
  return cuda_status(launch_f_impl(h->p, (const double2*)u, (double2*)fi, nb, (cudaStream_t)stream),
                     "sdcsw_f_impl");
}

int sdcsw_implicit_solve(sdcsw_plan* h, const double* coef, const double* beta, double* u, int nb,
                         void* stream) {
  int st = check_plan(h, 1, "sdcsw_implicit_solve");
  if (st) return st;
  if (nb < 0 || !coef) return SDCSW_ERR_PARAM;
  if (nb == 0) return SDCSW_OK;
  return cuda_status(launch_solve(h->p, coef, (const double2*)beta, (double2*)u, nb,
                                  (cudaStream_t)stream),
                     "sdcsw_implicit_solve");
}

int sdcsw_sweep_nodes(sdcsw_plan* h, int n_nodes, int node_lo, int count, const double* node_coef,
                      const double* u0, const double* fe, long long fe_stride, const double* fi,
                      long long fi_stride, int first, double* u_out, double* fi_out, void* stream) {
  int st = check_plan(h, 1, "sdcsw_sweep_nodes");
  if (st) return st;
  if (n_nodes < 1 || n_nodes > 16 || node_lo < 0 || count < 0 || node_lo + count > n_nodes ||
      !node_coef) {
    set_error("sdcsw_sweep_nodes: bad node range");
    return SDCSW_ERR_PARAM;
  }
  if (count == 0) return SDCSW_OK;
  return cuda_status(launch_sweep_nodes(h->p, n_nodes, node_lo, count, node_coef,
                                        (const double2*)u0, (const double2*)fe, fe_stride,
                                        (const double2*)fi, fi_stride, first, (double2*)u_out,
                                        (double2*)fi_out, nullptr, (cudaStream_t)stream),
                     "sdcsw_sweep_nodes");
}

int sdcsw_sweep_nodes_residual(sdcsw_plan* h, int n_nodes, int node_lo, int count,
                               const double* node_coef, const double* u0, const double* fe,
                               long long fe_stride, const double* fi, long long fi_stride, int first,
                               const double* u_prev, double* u_out, double* fi_out, double* resid,
                               void* stream) {
  int st = check_plan(h, 1, "sdcsw_sweep_nodes_residual");
  if (st) return st;
  if (n_nodes < 1 || n_nodes > kFuseMaxNodes || node_lo < 0 || count < 1 ||
      node_lo + count > n_nodes || !node_coef || !u_prev || !resid) {
    set_error("sdcsw_sweep_nodes_residual: bad node range (M <= 6) or null argument");
    return SDCSW_ERR_PARAM;
  }
  Plan& p = h->p;
  if (p.own_idx != nullptr) {
    set_error("sdcsw_sweep_nodes_residual: not available on a spectrally split plan");
    return SDCSW_ERR_STATE;
  }
  // the partials and the block counter are per plan: residual sweeps on one plan must be
  // serialised on one stream (include/sdcsw.h)
  const ResidArgs ra{u_prev, p.resid_part, p.resid_count, resid};
  return cuda_status(launch_sweep_nodes(p, n_nodes, node_lo, count, node_coef,
                                        (const double2*)u0, (const double2*)fe, fe_stride,
                                        (const double2*)fi, fi_stride, first, (double2*)u_out,
                                        (double2*)fi_out, nullptr, (cudaStream_t)stream, 1, 0, 0,
                                        0, nullptr, &ra),
                     "sdcsw_sweep_nodes_residual");
}

int sdcsw_final_node(sdcsw_plan* h, int n_nodes, const double* final_coef, const double* u0,
                     const double* fe, long long fe_stride, const double* fi, long long fi_stride,
                     int first, double* u_out, void* stream) {
  int st = check_plan(h, 1, "sdcsw_final_node");
  if (st) return st;
  if (n_nodes < 1 || n_nodes > 16 || !final_coef) return SDCSW_ERR_PARAM;
  return cuda_status(launch_final_node(h->p, n_nodes, final_coef, (const double2*)u0,
                                       (const double2*)fe, fe_stride, (const double2*)fi, fi_stride,
                                       first, (double2*)u_out, nullptr, nullptr, nullptr,
                                       (cudaStream_t)stream),
                     "sdcsw_final_node");
}

int sdcsw_serial_sweep(sdcsw_plan* h, int n_nodes, const double* coef, const double* u0,
                       const double* fe_old, long long fe_stride, const double* fi_old,
                       long long fi_stride, int first, double* fe_new, double* fi_new,
                       double* u_last, double* work, void* stream) {
  int st = check_plan(h, 1, "sdcsw_serial_sweep");
  if (st) return st;
  if ((st = check_spherical(h, "sdcsw_serial_sweep"))) return st;
  const int M = n_nodes;
  if (M < 1 || M > 16 || !coef || !u0 || !fe_old || !fi_old || !fe_new || !fi_new || !u_last ||
      !work) {
    set_error("sdcsw_serial_sweep: bad node count (1..16) or null argument");
    return SDCSW_ERR_PARAM;
  }
  Plan& p = h->p;
  if (p.own_idx != nullptr) {
    set_error("sdcsw_serial_sweep: not available on a spectrally split plan");
    return SDCSW_ERR_STATE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t S = (size_t)3 * p.C;
  const double* W = coef;             // [M][M]   dt q
  const double* we = W + M * M;       // [M]      dt explicit weights
  const double* wi = we + M;          // [M]      dt dtau
  const double* sc = wi + M;          // [M][3]   solve scalars
  double2* quad = reinterpret_cast<double2*>(work);  // [M] states
  double2* corr = quad + M * S;                      // [1]
  double2* ustage = corr + S;                        // [1]
  const double2* u = reinterpret_cast<const double2*>(u0);
  const double2* ofe = reinterpret_cast<const double2*>(fe_old);
  const double2* ofi = reinterpret_cast<const double2*>(fi_old);
  double2* nfe = reinterpret_cast<double2*>(fe_new);
  double2* nfi = reinterpret_cast<double2*>(fi_new);
  cudaError_t e = cudaSuccess;
  if (p.xsyn_nb != 1) {  // the API operand holds one state's records; padding rows zero
    e = cudaMemsetAsync(p.xsyn, 0, (size_t)p.rows * kXsyn * sizeof(double), s);
    p.xsyn_nb = 1;
  }
  // the serial branch of enqueue_step for one sweep (same kernels, same order)
  if (e == cudaSuccess)
    e = launch_serial_quad(p, M, W, u, ofe, fe_stride, ofi, fi_stride, first,
                           quad, s);
  for (int m = 0; m < M && e == cudaSuccess; ++m) {
    const bool last = m == M - 1;
    e = launch_serial_node(p, M, m, sc + 3 * m, quad + m * S, corr, u, ofi + fi_stride * m * S,
                           first, ustage, last ? reinterpret_cast<double2*>(u_last) : nullptr,
                           nfi + m * S, nullptr, nullptr, p.xsyn, s);
    if (e == cudaSuccess) e = f_expl_prepped(p, plan_work(p), p.xsyn, nfe + m * S, 1, s, nullptr);
    if (e == cudaSuccess && m + 1 < M)
      e = launch_serial_update(p, m, we[m], wi[m], corr, nfe + m * S, ofe + fe_stride * m * S,
                               nfi + m * S, ofi + fi_stride * m * S, u, first, s);
  }
  return cuda_status(e, "sdcsw_serial_sweep");
}

int sdcsw_transform_stage(sdcsw_plan* h, int stage, const double* in, double* out, int nb,
                          void* stream) {
  int st = check_plan(h, nb, "sdcsw_transform_stage");
  if (st) return st;
  if ((st = check_spherical(h, "sdcsw_transform_stage"))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  switch (stage) {
    case 0:
      if (h->p.xsyn_nb != nb) {
        e = cudaMemsetAsync(h->p.xsyn, 0, (size_t)h->p.rows * nb * kXsyn * sizeof(double), s);
        if (e != cudaSuccess) break;
        h->p.xsyn_nb = nb;
      }
      e = launch_synth_prep(h->p, (const double2*)in, nb, h->p.xsyn, s);
      if (e == cudaSuccess) e = launch_synthesis(h->p, plan_work(h->p), h->p.xsyn, nb, s, nullptr);
      break;
    // (H-free plans: stage 3 includes the operand conversion, stage 2 the assembly)
    case 3: e = launch_synthesis(h->p, plan_work(h->p), h->p.xsyn, nb, s, nullptr); break;
    case 1: e = launch_ring(h->p, plan_work(h->p), nb, s); break;
    case 2: e = launch_analysis(h->p, plan_work(h->p), (double2*)out, nb, s); break;
    case 4: {  // analysis with the fused node-update epilogue, as in the dSDC step (nb nodes)
      if (!fuse_supported(h->p, nb)) {
        set_error("sdcsw_transform_stage: no fused analysis for this plan / batch");
        return SDCSW_ERR_PARAM;
      }
      FuseArgs fz{};
      fz.mode = 1;
      fz.M = nb;
      fz.u0 = in;
      fz.fi = out;
      fz.xsyn = h->p.xsyn;
      fz.phibar = h->p.phibar;
      h->p.xsyn_nb = -1;  // the operand layout is overwritten
      e = launch_analysis_fused(h->p, plan_work(h->p), nb, fz, s);
      break;
    }
    default: set_error("sdcsw_transform_stage: stage must be 0..4"); return SDCSW_ERR_PARAM;
  }
  return cuda_status(e, "sdcsw_transform_stage");
}

int sdcsw_workspace(sdcsw_plan* h, int which, void** ptr, long long* bytes) {
  int st = check_plan(h, 1, "sdcsw_workspace");
  if (st) return st;
  if ((st = check_spherical(h, "sdcsw_workspace"))) return st;
  if (!ptr || !bytes || which < 0 || which > 1) return SDCSW_ERR_PARAM;
  const Plan& p = h->p;
  const long long per = (long long)p.max_batch * p.J * p.L * 2 * sizeof(double2);
  *ptr = which == 0 ? (void*)p.fsyn : (void*)p.gan;
  *bytes = which == 0 ? per * 4 : per * (ponly_on(p) ? kSlotsP : kNumSlots);  // see sdcsw.h
  return SDCSW_OK;
}

int sdcsw_plan_transform_kind(sdcsw_plan* h, int* kind, int* rows) {
  int st = check_plan(h, 1, "sdcsw_plan_transform_kind");
  if (st) return st;
  const Plan& p = h->p;
  const bool po = ponly_on(p);
  if (kind) *kind = po ? 1 : 0;
  if (rows) *rows = po ? p.rowsP : p.rows;
  return SDCSW_OK;
}

int sdcsw_plan_set_split(sdcsw_plan* h, int S, int sp, void* fourier, long long bytes) {
  int st = check_plan(h, 1, "sdcsw_plan_set_split");
  if (st) return st;
  if ((st = check_spherical(h, "sdcsw_plan_set_split"))) return st;
  Plan& p = h->p;
  if (S < 1 || sp < 0 || sp >= S || S > p.L) {
    set_error("sdcsw_plan_set_split: need 1 <= S <= T+1 and 0 <= sp < S");
    return SDCSW_ERR_PARAM;
  }
  cudaSetDevice(p.device);
  cudaDeviceSynchronize();
  for (int** q : {&p.m_part, &p.m_k, &p.own_m, &p.own_work, &p.own_idx, &p.own_workP}) {
    if (*q) dev_free(*q);
    *q = nullptr;
  }
  p.n_own_workP = 0;
  p.split_S = S;
  p.split_sp = sp;
  p.Lp = p.L;
  p.fsyn_ext = nullptr;
  p.n_own_m = p.L;
  p.n_own_work = p.n_own_idx = 0;
  if (S == 1) return SDCSW_OK;
  // pairs (m, T - m) dealt round-robin to the parts: equal coefficient counts
  const int T = p.T, L = p.L;
  std::vector<int> part(L), kpos(L), cnt(S, 0);
  for (int i = 0, m = 0; m <= T - m; ++m, ++i) {
    part[m] = i % S;
    part[T - m] = i % S;
  }
  std::vector<int> own;
  for (int m = 0; m < L; ++m) {
    kpos[m] = cnt[part[m]]++;
    if (part[m] == sp) own.push_back(m);
  }
  int Lp = 0;
  for (int q = 0; q < S; ++q) Lp = cnt[q] > Lp ? cnt[q] : Lp;
  const long long need = (long long)S * p.max_batch * p.J * Lp * 8 * sizeof(double2);
  if (!fourier || bytes < need) {
    set_error("sdcsw_plan_set_split: Fourier buffer smaller than S * max_batch * (nlat/2) * Lp * 128 B");
    return SDCSW_ERR_PARAM;
  }
  // own analysis work items and coefficient indices
  std::vector<int> work(p.n_anal_work), wown, idx;
  cudaMemcpy(work.data(), p.anal_work, work.size() * sizeof(int), cudaMemcpyDeviceToHost);
  for (int w : work)
    if (part[w >> 16] == sp) wown.push_back(w);
  std::vector<int> wownP;  // H-free analysis work items of own m
  if (p.anal_workP != nullptr) {
    std::vector<int> workP(p.n_anal_workP);
    cudaMemcpy(workP.data(), p.anal_workP, workP.size() * sizeof(int), cudaMemcpyDeviceToHost);
    for (int w : workP)
      if (part[w >> 16] == sp) wownP.push_back(w);
  }
  for (int m : own) {
    const int mo = m * (T + 1) - m * (m - 1) / 2;
    for (int n = m; n <= T; ++n) idx.push_back(mo + n - m);
  }
  cudaError_t e;
  if ((e = upload(&p.m_part, part.data(), part.size())) != cudaSuccess ||
      (e = upload(&p.m_k, kpos.data(), kpos.size())) != cudaSuccess ||
      (e = upload(&p.own_m, own.data(), own.size())) != cudaSuccess ||
      (e = upload(&p.own_work, wown.data(), wown.size())) != cudaSuccess ||
      (e = upload(&p.own_idx, idx.data(), idx.size())) != cudaSuccess ||
      (!wownP.empty() && (e = upload(&p.own_workP, wownP.data(), wownP.size())) != cudaSuccess))
    return cuda_status(e, "sdcsw_plan_set_split");
  p.n_own_workP = (int)wownP.size();
  p.Lp = Lp;
  p.n_own_m = (int)own.size();
  p.n_own_work = (int)wown.size();
  p.n_own_idx = (int)idx.size();
  p.fsyn_ext = (double2*)fourier;
  p.xsyn_nb = -1;  // the operand buffer is rebuilt for the own rows
  return SDCSW_OK;
}

int sdcsw_split_info(sdcsw_plan* h, int* Lp, int* n_own_m, int* n_own_idx) {
  int st = check_plan(h, 1, "sdcsw_split_info");
  if (st) return st;
  if ((st = check_spherical(h, "sdcsw_split_info"))) return st;
  if (Lp) *Lp = h->p.split_S > 1 ? h->p.Lp : 0;
  if (n_own_m) *n_own_m = h->p.n_own_m;
  if (n_own_idx) *n_own_idx = h->p.split_S > 1 ? h->p.n_own_idx : h->p.C;
  return SDCSW_OK;
}

int sdcsw_split_f_expl_begin(sdcsw_plan* h, const double* u, int nb, void* stream) {
  int st = check_plan(h, nb, "sdcsw_split_f_expl_begin");
  if (st) return st;
  if ((st = check_spherical(h, "sdcsw_split_f_expl_begin"))) return st;
  Plan& p = h->p;
  if (p.split_S < 2) {
    set_error("sdcsw_split_f_expl_begin: plan is not split");
    return SDCSW_ERR_STATE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (p.xsyn_nb != nb) {
    e = cudaMemsetAsync(p.xsyn, 0, (size_t)p.rows * nb * kXsyn * sizeof(double), s);
    p.xsyn_nb = nb;
  }
  if (e == cudaSuccess) e = launch_synth_prep(p, (const double2*)u, nb, p.xsyn, s);
  if (e == cudaSuccess) e = launch_synthesis_split(p, p.xsyn, nb, s);
  return cuda_status(e, "sdcsw_split_f_expl_begin");
}

int sdcsw_split_f_expl_end(sdcsw_plan* h, double* fe, int nb, void* stream) {
  int st = check_plan(h, nb, "sdcsw_split_f_expl_end");
  if (st) return st;
  if ((st = check_spherical(h, "sdcsw_split_f_expl_end"))) return st;
  const Plan& p = h->p;
  if (p.split_S < 2) {
    set_error("sdcsw_split_f_expl_end: plan is not split");
    return SDCSW_ERR_STATE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_ring_split(p, plan_work(p), nb, s);
  if (e == cudaSuccess) e = launch_analysis(p, plan_work(p), (double2*)fe, nb, s);
  return cuda_status(e, "sdcsw_split_f_expl_end");
}

int sdcsw_axpy(long long n, const double* x, double w, const double* y, double* out, void* stream) {
  if (n < 0 || !x || !y || !out) return SDCSW_ERR_PARAM;
  if (n == 0) return SDCSW_OK;
  return cuda_status(launch_axpy(n, x, w, y, out, (cudaStream_t)stream), "sdcsw_axpy");
}

int sdcsw_check_finite(const double* x, long long n, int* flag, void* stream) {
  if (n < 0 || !flag) return SDCSW_ERR_PARAM;
  if (n == 0) return SDCSW_OK;
  return cuda_status(launch_check_finite(x, n, flag, (cudaStream_t)stream), "sdcsw_check_finite");
}

// ---------------------------------------------------------------------------
// stepper
// ---------------------------------------------------------------------------
static bool serial_fused_active(const sdcsw_stepper* st) {
  return st->fuse && st->mode == 1 && st->members == 1 && fuse_supported(st->plan->p, st->M);
}

static bool fused_active(const sdcsw_stepper* st) {
  return st->fuse && st->mode == 0 && st->members == 1 && st->chains == 1 && !st->sequential &&
         fuse_supported(st->plan->p, st->M);
}

// dSDC with every node update in the epilogue of the analysis that produced
// its f_E operands: K x (synthesis -> ring -> fused analysis).  f_I of the
// nodes is updated in place (a thread owns one element for all nodes).
static cudaError_t enqueue_step_fused(sdcsw_stepper* st, double2* u, cudaStream_t s) {
  const Plan& p = st->plan->p;
  const int M = st->M, K = st->K;
  const int cstride = M * (M + 4);
  FuseArgs fz{};
  fz.M = M;
  fz.u0 = reinterpret_cast<const double*>(u);
  fz.fi = reinterpret_cast<double*>(st->fi);
  fz.u_out = reinterpret_cast<double*>(u);
  fz.diverged = st->flags;
  fz.step_counter = st->flags + 1;
  fz.phibar = p.phibar;
  const Work w = plan_work(p);
  for (int k = 1; k <= K; ++k) {
    const int nb = k == 1 ? 1 : M;
    cudaError_t e = launch_synthesis(p, w, k == 1 ? st->xsyn1 : st->xsynM, nb, s,
                                     k == 1 ? st->flags + 1 : nullptr);
    if (e != cudaSuccess) return e;
    if ((e = launch_ring(p, w, nb, s)) != cudaSuccess) return e;
    fz.first = k == 1;
    fz.mode = k < K ? 1 : 2;
    fz.xsyn = k < K ? st->xsynM : st->xsyn1;
    const double* c = st->coef.data() + (size_t)(k - 1) * cstride;
    const int nc = k < K ? cstride : M + 4;
    for (int q = 0; q < nc; ++q) fz.cf[q] = c[q];
    if ((e = launch_analysis_fused(p, w, nb, fz, s)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// serial SDC with serial_update(m) and serial_node(m + 1) in the epilogue of
// node m's analysis: per sweep quad + node 0 + M x (synthesis, ring, analysis)
static cudaError_t enqueue_serial_fused(sdcsw_stepper* st, double2* u, cudaStream_t s) {
  const Plan& p = st->plan->p;
  const int M = st->M, K = st->K;
  const size_t S = st->S;
  int* diverged = st->flags;
  int* counter = st->flags + 1;
  const double* W = st->coef.data();
  const double* we = W + M * M;
  const double* wi = we + M;
  const double* sc = wi + M;
  const Work w = plan_work(p);
  cudaError_t e = f_expl_prepped(p, w, st->xsyn1, st->fe0, 1, s, counter, 0);
  if (e != cudaSuccess) return e;
  double2* old_fe = st->fe0;
  double2* old_fi = st->fi;
  long long old_stride = 0;
  int first = 1;
  auto D = [](const double2* q) { return reinterpret_cast<const double*>(q); };
  auto Wr = [](double2* q) { return reinterpret_cast<double*>(q); };
  for (int k = 1; k <= K; ++k) {
    double2* nfe = (k % 2) ? st->fe : st->feB;
    double2* nfi = (k % 2) ? st->fi : st->fiB;
    if ((e = launch_serial_quad(p, M, W, u, old_fe, old_stride, old_fi, old_stride, first,
                                st->quad, s)) != cudaSuccess)
      return e;
    const bool last0 = k == K && M == 1;
    if ((e = launch_serial_node(p, M, 0, sc, st->quad, st->corr, u, old_fi, first, st->ustage,
                                last0 ? u : nullptr, nfi, last0 ? diverged : nullptr,
                                last0 ? counter : nullptr, st->xsyn1, s)) != cudaSuccess)
      return e;
    for (int m = 0; m < M; ++m) {
      if ((e = launch_synthesis(p, w, st->xsyn1, 1, s, nullptr)) != cudaSuccess) return e;
      if ((e = launch_ring(p, w, 1, s)) != cudaSuccess) return e;
      FuseArgs fz{};
      fz.mode = 3;
      fz.M = M;
      fz.first = first;
      fz.u0 = D(u);
      fz.phibar = p.phibar;
      fz.xsyn = st->xsyn1;
      fz.fe_new = Wr(nfe + m * S);
      fz.fe_old = D(old_fe + old_stride * m * S);
      fz.fi_old = D(old_fi + old_stride * m * S);
      fz.fi_new = D(nfi + m * S);
      fz.corr = Wr(st->corr);
      fz.use_corr = m > 0;
      if (m + 1 < M) {
        const bool last = k == K && m + 1 == M - 1;
        fz.quad_next = D(st->quad + (m + 1) * S);
        fz.fi_old_next = D(old_fi + old_stride * (m + 1) * S);
        fz.fi_new_next = Wr(nfi + (m + 1) * S);
        fz.u_out = last ? Wr(u) : nullptr;
        fz.diverged = last ? diverged : nullptr;
        fz.step_counter = last ? counter : nullptr;
        fz.cf[0] = we[m];
        fz.cf[1] = wi[m];
        for (int q = 0; q < 3; ++q) fz.cf[2 + q] = sc[3 * (m + 1) + q];
      }
      if ((e = launch_analysis_fused(p, w, 1, fz, s)) != cudaSuccess) return e;
    }
    old_fe = nfe;
    old_fi = nfi;
    old_stride = 1;
    first = 0;
  }
  return cudaSuccess;
}

static cudaError_t enqueue_step(sdcsw_stepper* st, double2* u, cudaStream_t s,
                                cudaEvent_t* marks = nullptr) {
  if (marks == nullptr && fused_active(st)) return enqueue_step_fused(st, u, s);
  if (marks == nullptr && serial_fused_active(st)) return enqueue_serial_fused(st, u, s);
  const Plan& p = st->plan->p;
  const int M = st->M, K = st->K;
  const size_t S = st->S;
  int* diverged = st->flags;
  int* counter = st->flags + 1;
  // f_E(u0) of every member from the operand the previous step's last kernel
  // (or the run's prep) wrote into xsyn1
  const int E = st->members;
  if (marks) cudaEventRecord(marks[0], s);
  const bool planar = p.kind == 1;  // planar: f_E reads the node states, no operand records
  const bool sprep = st->sprep && st->mode == 0;  // H-free: f_E from the node states too
  cudaError_t e = planar  ? planar_f_expl(p, u, st->fe0, E, s, counter)
                  : sprep ? f_expl_states_ponly(p, plan_work(p), u, st->fe0, E, s, counter)
                          : f_expl_prepped(p, plan_work(p), st->xsyn1, st->fe0, E, s, counter,
                                           p.fe_chunk);
  if (e != cudaSuccess) return e;
  if (marks) cudaEventRecord(marks[1], s);
  if (st->mode == 0) {
    // fe and fi alternate between two buffers: every node reads all fe_j, fi_j
    // of the previous sweep while its own new values are written (by a
    // concurrent chain, or by an earlier node in sequential mode).  The M node
    // updates of a sweep are independent (the paper's parallel-across-the-
    // method structure): they run as `chains` concurrent graph branches, each
    // a contiguous node group doing solve -> synthesis -> ring -> analysis.
    // Tendency buffers are member-major [E][M]; an ensemble runs as one chain
    // whose GEMMs carry all E * M states as columns.
    const int cstride = M * (M + 4);
    const int G = st->sequential ? M : st->chains;
    const bool seq = st->sequential != 0;  // groups of one node, all on stream s
    const long long mS = M;  // member stride of the node buffers, in states
    double2* fi_cur = st->fi;
    double2* fe_cur = st->fe0;
    for (int k = 1; k < K; ++k) {
      const bool first = k == 1;
      double2* fi_new = (k % 2) ? st->fi : st->fiB;
      double2* fe_new = (k % 2) ? st->fe : st->feB;
      const double* coef = st->coef.data() + (size_t)(k - 1) * cstride;
      if (G > 1 && !seq) {
        if ((e = cudaEventRecord(st->ev_fork, s)) != cudaSuccess) return e;
        for (int g = 0; g < G; ++g)
          if ((e = cudaStreamWaitEvent(st->side[g], st->ev_fork, 0)) != cudaSuccess) return e;
      }
      for (int g = 0; g < G; ++g) {
        const int lo = g * M / G, hi = (g + 1) * M / G, cnt = hi - lo;
        cudaStream_t sg = (G > 1 && !seq) ? st->side[g] : s;
        if (sprep && st->nodes_po) {  // H-free: the node kernel writes the P-only operand
          // into the stepper's own operand storage (zeroed at creation, written only here,
          // always with this group's layout: its padding rows stay zero)
          double* xo = st->xsynM + (size_t)lo * E * p.rowsP * kXsynP;
          e = launch_sweep_nodes_po(p, M, lo, cnt, coef, u, fe_cur, first ? 0 : 1, fi_cur,
                                    first ? 0 : 1, first, fi_new + lo * S, xo, sg, E,
                                    first ? 1 : mS, mS);
          if (e != cudaSuccess) return e;
          e = f_expl_operand_ponly(p, plan_work(p, lo), xo, fe_new + lo * S, cnt * E, sg);
          if (e != cudaSuccess) return e;
          continue;
        }
        const bool keep = planar || sprep;  // node states stored for an f_E that reads them
        double* xs = keep ? nullptr : st->xsynM + (size_t)lo * E * p.rows * kXsyn;
        // spherical P/H: the node states reach the f_E only as synthesis operands (xs),
        // so they are not stored; the planar and H-free f_E read them from ustage
        e = launch_sweep_nodes(p, M, lo, cnt, coef, u, fe_cur, first ? 0 : 1,
                               fi_cur, first ? 0 : 1, first, keep ? st->ustage + lo * S : nullptr,
                               fi_new + lo * S, xs, sg, E, first ? 1 : mS, mS, p.fe_chunk);
        if (e != cudaSuccess) return e;
        e = planar  ? planar_f_expl(p, st->ustage + lo * S, fe_new + lo * S, cnt * E, sg, nullptr)
            : sprep ? f_expl_states_ponly(p, plan_work(p, lo), st->ustage + lo * S, fe_new + lo * S,
                                          cnt * E, sg, nullptr)
                    : f_expl_prepped(p, plan_work(p, lo), xs, fe_new + lo * S, cnt * E, sg,
                                     nullptr, p.fe_chunk);
        if (e != cudaSuccess) return e;
      }
      if (G > 1 && !seq) {
        for (int g = 0; g < G; ++g) {
          if ((e = cudaEventRecord(st->ev_join[g], st->side[g])) != cudaSuccess) return e;
          if ((e = cudaStreamWaitEvent(s, st->ev_join[g], 0)) != cudaSuccess) return e;
        }
      }
      if (marks) cudaEventRecord(marks[1 + k], s);
      if (marks && st->hook) {  // host callback after sweep k (device idle meanwhile)
        if ((e = cudaEventSynchronize(marks[1 + k])) != cudaSuccess) return e;
        st->hook(st->hook_user, k);
      }
      fi_cur = fi_new;
      fe_cur = fe_new;
    }
    const bool first = K == 1;
    double* xs1 = planar || sprep ? nullptr : st->xsyn1;
    if (marks) {
      e = launch_final_node(p, M, st->coef.data() + (size_t)(K - 1) * cstride, u,
                            fe_cur, first ? 0 : 1, fi_cur, first ? 0 : 1,
                            first, u, diverged, counter, xs1, s, E, first ? 1 : mS, mS);
      cudaEventRecord(marks[K + 1], s);
      return e;
    }
    return launch_final_node(p, M, st->coef.data() + (size_t)(K - 1) * cstride, u,
                             fe_cur, first ? 0 : 1, fi_cur, first ? 0 : 1,
                             first, u, diverged, counter, xs1, s, E, first ? 1 : mS, mS);
  }
  // serial SDC: old/new tendency buffers alternate between sweeps
  const double* W = st->coef.data();
  const double* we = W + M * M;
  const double* wi = we + M;
  const double* sc = wi + M;
  double2* old_fe = st->fe0;
  double2* old_fi = st->fi;
  long long old_stride = 0;
  int first = 1;
  for (int k = 1; k <= K; ++k) {
    double2* nfe = (k % 2) ? st->fe : st->feB;
    double2* nfi = (k % 2) ? st->fi : st->fiB;
    e = launch_serial_quad(p, M, W, u, old_fe, old_stride, old_fi, old_stride, first, st->quad, s);
    if (e != cudaSuccess) return e;
    for (int m = 0; m < M; ++m) {
      const bool last = (k == K && m == M - 1);
      e = launch_serial_node(p, M, m, sc + 3 * m, st->quad + m * S, st->corr, u,
                             old_fi + old_stride * m * S, first, st->ustage, last ? u : nullptr,
                             nfi + m * S, last ? diverged : nullptr, last ? counter : nullptr,
                             planar ? nullptr : st->xsyn1, s);
      if (e != cudaSuccess) return e;
      e = planar ? planar_f_expl(p, st->ustage, nfe + m * S, 1, s, nullptr)
                 : f_expl_prepped(p, plan_work(p), st->xsyn1, nfe + m * S, 1, s, nullptr);
      if (e != cudaSuccess) return e;
      if (m + 1 < M) {
        e = launch_serial_update(p, m, we[m], wi[m], st->corr, nfe + m * S,
                                 old_fe + old_stride * m * S, nfi + m * S,
                                 old_fi + old_stride * m * S, u, first, s);
        if (e != cudaSuccess) return e;
      }
    }
    old_fe = nfe;
    old_fi = nfi;
    old_stride = 1;
    first = 0;
    if (marks) cudaEventRecord(marks[1 + k], s);
    if (marks && st->hook) {
      if ((e = cudaEventSynchronize(marks[1 + k])) != cudaSuccess) return e;
      st->hook(st->hook_user, k);
    }
  }
  return cudaSuccess;
}

int sdcsw_stepper_create(sdcsw_plan* h, int mode, int n_nodes, int n_sweeps, const double* coef,
                         int n_coef, sdcsw_stepper** out) {
  return sdcsw_stepper_create_ensemble(h, mode, n_nodes, n_sweeps, 1, coef, n_coef, out);
}

int sdcsw_stepper_create_ensemble(sdcsw_plan* h, int mode, int n_nodes, int n_sweeps, int members,
                                  const double* coef, int n_coef, sdcsw_stepper** out) {
  int st = check_plan(h, 1, "sdcsw_stepper_create");
  if (st) return st;
  const int M = n_nodes, K = n_sweeps, E = members;
  if ((mode != 0 && mode != 1) || M < 1 || M > 16 || K < 1 || !coef || !out || E < 1 ||
      (mode == 1 && E != 1) || E > 65535) {
    set_error("sdcsw_stepper_create: bad mode / node / sweep / member count");
    return SDCSW_ERR_PARAM;
  }
  const int want = mode == 0 ? K * M * (M + 4) : M * M + 2 * M + 3 * M;
  const int need = mode == 0 ? (K - 1) * M * (M + 4) + (M + 4) : want;
  if (n_coef < need) {
    set_error("sdcsw_stepper_create: coefficient array too short");
    return SDCSW_ERR_PARAM;
  }
  if (h->p.split_S > 1) {
    set_error("sdcsw_stepper_create: plan is spectrally split (use the node/spectral orchestration)");
    return SDCSW_ERR_STATE;
  }
  if (mode == 0 && M * E > h->p.max_batch) {
    set_error("sdcsw_stepper_create: plan max_batch < nodes x members");
    return SDCSW_ERR_PARAM;
  }
  sdcsw_stepper* s = new (std::nothrow) sdcsw_stepper();
  if (!s) return SDCSW_ERR_PARAM;
  s->plan = h; s->mode = mode; s->M = M; s->K = K; s->members = E;
  s->coef.assign(coef, coef + need);
  if (mode == 0) {
    // pad: final block stored at index K-1
    s->coef.resize((size_t)K * M * (M + 4), 0.0);
    const size_t fin = (size_t)(K - 1) * M * (M + 4);
    std::vector<double> tail(coef + (size_t)(K - 1) * M * (M + 4), coef + need);
    for (size_t q = 0; q < tail.size(); ++q) s->coef[fin + q] = tail[q];
  }
  const Plan& p = h->p;
  s->S = (size_t)3 * p.C;
  // sweep storage per member: fe0, and fe / fi of the nodes twice (the sweep
  // that is read and the one being written: the node updates of a sweep run
  // concurrently and every one reads all old tendencies); node states only
  // where an f_E reads them (planar dSDC; one state for serial SDC) - the
  // spherical dSDC step keeps node states only as synthesis operands
  // H-free plans (legendre_ponly.cu): the dSDC step keeps its node states and builds the
  // P-only synthesis operand from them (k_prep_ponly), instead of writing 12-double
  // operand records that a conversion kernel re-reads (c4: -100 MB per f_E of 256 states)
  const int sprep = mode == 0 && p.kind == 0 && ponly_on(p) && p.own_idx == nullptr ? 1 : 0;
  // and with M <= kFuseMaxNodes the sweep's node kernel writes that operand directly
  // (k_sweep_nodes_po: no node states, no operand kernel; SDCSW_NODES_PO=0 turns it off)
  int nodes_po = sprep && M <= kFuseMaxNodes ? 1 : 0;
  if (const char* env = getenv("SDCSW_NODES_PO")) nodes_po = nodes_po && atoi(env) != 0;
  const size_t ust = mode == 1 ? 1 : (p.kind == 1 || (sprep && !nodes_po) ? (size_t)E * M : 0);
  const size_t nstates = (size_t)E * (1 + 4 * (size_t)M) + ust + (mode == 1 ? (size_t)M + 1 : 0);
  s->nstates = nstates;
  cudaError_t e = cudaSetDevice(p.device);
  if (e == cudaSuccess) e = dev_alloc(&s->buf, nstates * s->S * sizeof(double2));
  if (e == cudaSuccess) e = dev_alloc(&s->flags, 2 * sizeof(int));
  // operand records per state: 12-double rows, or (H-free sweeps) 8-double P-only rows
  const size_t xs = std::max((size_t)p.rows * kXsyn, (size_t)p.rowsP * kXsynP) * sizeof(double);
  if (e == cudaSuccess) e = dev_alloc(&s->xsyn1, xs * E * (1 + M));
  if (e == cudaSuccess) e = cudaMemset(s->xsyn1, 0, xs * E * (1 + M));
  s->xsynM = s->xsyn1 ? s->xsyn1 + xs / sizeof(double) * E : nullptr;
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    if (s->buf) dev_free(s->buf);
    if (s->flags) dev_free(s->flags);
    if (s->xsyn1) dev_free(s->xsyn1);
    delete s;
    return cuda_status(e, "sdcsw_stepper_create");
  }
  cudaMemset(s->buf, 0, nstates * s->S * sizeof(double2));
  double2* q = s->buf;
  s->fe0 = q; q += E * s->S;
  s->fe = q; q += E * M * s->S;
  s->fi = q; q += E * M * s->S;
  s->ustage = ust ? q : nullptr; q += ust * s->S;
  s->sprep = sprep;
  s->nodes_po = nodes_po;
  s->fiB = q; q += E * M * s->S;
  s->feB = q; q += E * M * s->S;
  if (mode == 1) {
    s->quad = q; q += M * s->S;
    s->corr = q; q += s->S;
  }
  const int init[2] = {INT_MAX, 0};
  cudaMemcpy(s->flags, init, sizeof(init), cudaMemcpyHostToDevice);
  // concurrent node chains: small truncations are latency-bound (one chain per
  // node fills the GPU); large ones batch all nodes through the GEMMs (table
  // reuse).  SDCSW_CHAINS overrides.
  s->chains = 1;
  s->fuse = E == 1 && fuse_supported(p, M);
  if (const char* env = getenv("SDCSW_FUSE")) s->fuse = s->fuse && atoi(env) != 0;
  if (mode == 0) {
    s->chains = (p.kind == 0 && p.T < 200 && E == 1 && !s->fuse) ? (M < 2 ? M : 2) : 1;
    if (const char* env = getenv("SDCSW_CHAINS")) s->chains = atoi(env);
    if (s->chains < 1) s->chains = 1;
    if (s->chains > M) s->chains = M;
    if (E > 1 || p.kind == 1) s->chains = 1;  // planar f_E shares one workspace
  }
  s->ncreated = mode == 0 && E == 1 && p.kind == 0 ? M : 0;  // side streams for up to M chains
  if (s->ncreated > 1) {
    cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming);
    for (int g = 0; g < s->ncreated; ++g) {
      cudaStreamCreateWithFlags(&s->side[g], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&s->ev_join[g], cudaEventDisableTiming);
    }
  }
  // several steps per replayed graph: PDL then also overlaps the step boundaries
  s->graph_steps = 8;
  if (const char* env = getenv("SDCSW_GRAPH_STEPS")) s->graph_steps = atoi(env) > 0 ? atoi(env) : 1;
  sdcsw_stepper_launches_per_step(s, &s->launches);
  *out = s;
  return SDCSW_OK;
}

static void drop_graphs(sdcsw_stepper* s) {
  if (s->exec) { cudaGraphExecDestroy(s->exec); s->exec = nullptr; }
  if (s->graph) { cudaGraphDestroy(s->graph); s->graph = nullptr; }
  if (s->execK) { cudaGraphExecDestroy(s->execK); s->execK = nullptr; }
  if (s->graphK) { cudaGraphDestroy(s->graphK); s->graphK = nullptr; }
}

int sdcsw_stepper_destroy(sdcsw_stepper* s) {
  if (!s) return SDCSW_ERR_STATE;
  cudaSetDevice(s->plan->p.device);
  cudaDeviceSynchronize();
  drop_graphs(s);
  if (s->ncreated > 1) {
    cudaEventDestroy(s->ev_fork);
    for (int g = 0; g < s->ncreated; ++g) {
      cudaStreamDestroy(s->side[g]);
      cudaEventDestroy(s->ev_join[g]);
    }
  }
  if (s->prof_ready)
    for (int i = 0; i < s->K + 2; ++i) cudaEventDestroy(s->prof[i]);
  cudaStreamDestroy(s->cap);
  dev_free(s->buf);
  dev_free(s->flags);
  dev_free(s->xsyn1);
  delete s;
  return SDCSW_OK;
}

int sdcsw_stepper_reset(sdcsw_stepper* s, void* stream) {
  if (!s) return SDCSW_ERR_STATE;
  const int init[2] = {INT_MAX, 0};
  return cuda_status(cudaMemcpyAsync(s->flags, init, sizeof(init), cudaMemcpyHostToDevice,
                                     (cudaStream_t)stream),
                     "sdcsw_stepper_reset");
}

int sdcsw_stepper_launches_per_step(sdcsw_stepper* s, int* n) {
  if (!s || !n) return SDCSW_ERR_STATE;
  const int G = s->sequential ? s->M : s->chains;
  s->launches = s->mode == 0 ? (fused_active(s) ? 3 * s->K : 4 + 4 * G * (s->K - 1))
                             : (serial_fused_active(s) ? 3 + s->K * (2 + 3 * s->M)
                                                       : 3 + s->K * 5 * s->M);
  // H-free plans: every f_E adds its operand kernel (prep or conversion) and the assembly;
  // with nodes_po the sweeps' operand comes from the node kernel (assembly only)
  if (ponly_on(s->plan->p) && !fused_active(s) && !serial_fused_active(s))
    s->launches += s->mode == 0 ? 2 + (s->nodes_po ? 1 : 2) * G * (s->K - 1) : 2 * (1 + s->K * s->M);
  *n = s->launches;
  return SDCSW_OK;
}

int sdcsw_stepper_run(sdcsw_stepper* s, double* u, int n_steps, int use_graph, void* stream) {
  if (!s || !u) {
    set_error("sdcsw_stepper_run: invalid handle or state");
    return SDCSW_ERR_STATE;
  }
  if (n_steps < 0) return SDCSW_ERR_PARAM;
  cudaStream_t cs = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(s->plan->p.device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  if (n_steps == 0) return SDCSW_OK;
  // the caller may have changed u since the last step: rebuild its synthesis operand
  // (H-free dSDC builds it from u inside every step)
  if (s->plan->p.kind == 0 && !s->sprep) {
    e = launch_synth_prep(s->plan->p, (const double2*)u, s->members, s->xsyn1, cs,
                          s->plan->p.fe_chunk);
    if (e != cudaSuccess) return cuda_status(e, "sdcsw_stepper_run prep");
  }
  if (!use_graph) {
    for (int i = 0; i < n_steps; ++i) {
      e = enqueue_step(s, (double2*)u, cs);
      if (e != cudaSuccess) return cuda_status(e, "sdcsw_stepper_run");
    }
    return SDCSW_OK;
  }
  if (!s->exec || s->graph_u != u) {
    drop_graphs(s);
    auto capture = [&](int steps, cudaGraph_t* g, cudaGraphExec_t* x) -> int {
      cudaError_t ce = cudaStreamBeginCapture(s->cap, cudaStreamCaptureModeThreadLocal);
      if (ce != cudaSuccess) return cuda_status(ce, "cudaStreamBeginCapture");
      cudaError_t le = cudaSuccess;
      for (int i = 0; i < steps && le == cudaSuccess; ++i) le = enqueue_step(s, (double2*)u, s->cap);
      ce = cudaStreamEndCapture(s->cap, g);
      if (le != cudaSuccess) return cuda_status(le, "capture step");
      if (ce != cudaSuccess) return cuda_status(ce, "cudaStreamEndCapture");
      ce = cudaGraphInstantiate(x, *g, 0);
      return ce == cudaSuccess ? SDCSW_OK : cuda_status(ce, "cudaGraphInstantiate");
    };
    int st = capture(1, &s->graph, &s->exec);
    if (st == SDCSW_OK && s->graph_steps > 1) st = capture(s->graph_steps, &s->graphK, &s->execK);
    if (st != SDCSW_OK) return st;
    s->graph_u = u;
  }
  int i = 0;
  if (s->execK)
    for (; i + s->graph_steps <= n_steps; i += s->graph_steps) {
      e = cudaGraphLaunch(s->execK, cs);
      if (e != cudaSuccess) return cuda_status(e, "cudaGraphLaunch");
    }
  for (; i < n_steps; ++i) {
    e = cudaGraphLaunch(s->exec, cs);
    if (e != cudaSuccess) return cuda_status(e, "cudaGraphLaunch");
  }
  return SDCSW_OK;
}

int sdcsw_stepper_set_option(sdcsw_stepper* s, int option, int value) {
  if (!s) return SDCSW_ERR_STATE;
  if (option == 0) {  // concurrent node chains
    if (value < 1 || value > s->M || (value > 1 && s->ncreated < value)) return SDCSW_ERR_PARAM;
    s->chains = value;
  } else if (option == 1) {  // sequential node updates
    if (s->mode != 0 || s->members != 1) return SDCSW_ERR_PARAM;
    s->sequential = value ? 1 : 0;
  } else if (option == 3) {  // steps per replayed graph
    if (value < 1 || value > 64) return SDCSW_ERR_PARAM;
    s->graph_steps = value;
  } else if (option == 2) {  // node updates fused into the analysis epilogue
    if (value && (s->members != 1 || !fuse_supported(s->plan->p, s->M)))
      return SDCSW_ERR_PARAM;
    s->fuse = value ? 1 : 0;
  } else {
    return SDCSW_ERR_PARAM;
  }
  drop_graphs(s);
  return SDCSW_OK;
}

int sdcsw_stepper_profile(sdcsw_stepper* s, double* u, double* stage_ms, int n, void* stream) {
  if (!s || !u || !stage_ms || n < s->K + 1) return SDCSW_ERR_PARAM;
  cudaStream_t cs = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(s->plan->p.device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  if (!s->prof_ready) {
    for (int i = 0; i < s->K + 2; ++i) cudaEventCreate(&s->prof[i]);
    s->prof_ready = true;
  }
  if (s->plan->p.kind == 0 && !s->sprep)
    e = launch_synth_prep(s->plan->p, (const double2*)u, s->members, s->xsyn1, cs,
                          s->plan->p.fe_chunk);
  if (e == cudaSuccess) e = enqueue_step(s, (double2*)u, cs, s->prof);
  if (e != cudaSuccess) return cuda_status(e, "sdcsw_stepper_profile");
  e = cudaEventSynchronize(s->prof[s->mode == 0 ? s->K + 1 : s->K]);
  if (e != cudaSuccess) return cuda_status(e, "sdcsw_stepper_profile");
  // stage_ms = [init, sweep_1 .. sweep_{K-1 or K}, final (dSDC)]
  const int nstages = s->mode == 0 ? s->K + 1 : s->K + 1;
  for (int i = 0; i < nstages; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->prof[i], s->prof[i + 1]);
    stage_ms[i] = ms;
  }
  return SDCSW_OK;
}

int sdcsw_stepper_step_hooked(sdcsw_stepper* s, double* u, sdcsw_sweep_hook hook, void* user,
                              double* stage_ms, int n, void* stream) {
  if (!s || !u || (stage_ms && n < s->K + 1)) return SDCSW_ERR_PARAM;
  if (s->members != 1) {
    set_error("sdcsw_stepper_step_hooked: one member only");
    return SDCSW_ERR_PARAM;
  }
  double local[42];
  s->hook = hook;
  s->hook_user = user;
  const int st = sdcsw_stepper_profile(s, u, stage_ms ? stage_ms : local, s->K + 1, stream);
  s->hook = nullptr;
  s->hook_user = nullptr;
  return st;
}

int sdcsw_stepper_sweep_state(sdcsw_stepper* s, int sweep, void** fe0, void** fe, void** fi) {
  if (!s || sweep < 1 || sweep > s->K) return SDCSW_ERR_PARAM;
  if (fe0) *fe0 = s->fe0;
  if (fe) *fe = (sweep % 2) ? s->fe : s->feB;
  if (fi) *fi = (sweep % 2) ? s->fi : s->fiB;
  return SDCSW_OK;
}

int sdcsw_stepper_storage(sdcsw_stepper* s, long long* bytes, long long* state_buffers) {
  if (!s) return SDCSW_ERR_STATE;
  const Plan& p = s->plan->p;
  const long long rec = (long long)std::max((size_t)p.rows * kXsyn, (size_t)p.rowsP * kXsynP) * sizeof(double);
  const long long ops = p.kind == 0 ? rec * s->members * (1 + s->M) : 0;
  if (bytes) *bytes = (long long)(s->nstates * s->S * sizeof(double2)) + ops + 2 * (long long)sizeof(int);
  if (state_buffers) *state_buffers = (long long)s->nstates;
  return SDCSW_OK;
}

int sdcsw_stepper_diverged(sdcsw_stepper* s, int* step_index) {
  if (!s || !step_index) return SDCSW_ERR_STATE;
  int v[2];
  cudaSetDevice(s->plan->p.device);
  cudaDeviceSynchronize();
  cudaError_t e = cudaMemcpy(v, s->flags, sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "sdcsw_stepper_diverged");
  *step_index = v[0] == INT_MAX ? 0 : v[0];
  return SDCSW_OK;
}

}  // extern "C"
