// Node-parallel dSDC over peer memory (include/sdcsw.h, sdcsw_exchange_*).
//
// The reference runs the M independent node updates of a diagonal sweep on a
// thread pool and joins them with a barrier before the next sweep
// (pkg/src/parsdc/integrators.py:254-288); every node's beta then reads all
// F_j = fe_j + fi_j.  Across GPUs (one process per GPU) rank r owns a
// contiguous node block, and the one exchange per sweep is done by the
// kernels themselves:
//
//   node kernel  (waits for the previous exchange, reads every node's fe, fi
//                 from the local exchange buffer, solves own nodes)
//   synthesis -> ring -> analysis  (own nodes; the analysis epilogue stores
//                 f_E and f_I of own nodes into every rank's buffer through
//                 NVLink - FuseArgs mode 4 - tile by tile as they are formed)
//   (the next consumer first posts the exchange number into every rank's
//    flag word, then waits until every rank has posted it)
//
// and after the last exchange every rank computes the closing solve and the
// next f_E(u0) redundantly (no further communication; the state stays
// replicated and bit-identical to the single-GPU stepper because every node
// kernel and transform is batch-invariant).  Protocol and buffer layout:
// internal.cuh (PeerFlags, PeerWait).
#include <climits>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "node_math.cuh"

namespace sdcsw {

struct PeerBases {
  double* x[kMaxPeers];  // exchange buffer of every rank q
};

// Copy-kernel publish (plans without the fused epilogue: T >= 400 TMA
// analysis): own nodes' fe (from a plain analysis) and fi into parity n & 1
// of every rank's buffer.  grid (ceil(S / 256), count)
__global__ void __launch_bounds__(256) k_peer_publish(long long S, int M, int lo,
                                                      const double2* __restrict__ fe_loc,
                                                      const double2* __restrict__ fi_loc,
                                                      const int* epoch, int k, int kx,
                                                      PeerBases pb, int world) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int b = blockIdx.y;
  const long long par = (long long)(exchange_number(epoch, k, kx) & 1);
  const double2 e = fe_loc[(size_t)b * S + i];
  const double2 f = fi_loc[(size_t)b * S + i];
  const size_t slot = ((size_t)par * M + lo + b) * 2 * S;  // in double2
  for (int q = 0; q < world; ++q) {
    double2* X = reinterpret_cast<double2*>(pb.x[q]);
    X[slot + i] = e;
    X[slot + S + i] = f;
  }
}

// Post only: a rank without nodes publishes nothing but still posts every
// exchange of the step (the closing solve posts and waits for the last one).
__global__ void k_peer_post(PeerWait pw) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  if (threadIdx.x == 0) {
    const unsigned long long n = exchange_number(pw.epoch, pw.k, pw.kx);
    for (int q = 0; q < pw.world; ++q) atomicMax_system(pw.post[q], n);
  }
}

}  // namespace sdcsw

using namespace sdcsw;

struct sdcsw_exchange {
  sdcsw_plan* plan;
  int M, K, world, rank, lo, count;
  std::vector<double> coef;  // K blocks of M (M + 4); block K-1 = final (M + 4)
  size_t S;                  // one state, in double2
  char* mem;                 // exchange buffer + control block (the IPC allocation)
  double2* X;                // [2][M][2][S]
  PeerFlags* pflag;          // flag block (after X in the IPC allocation)
  char* local;               // private buffers
  double2 *fe0, *fe_loc, *fi_loc;
  double *xsyn1, *xsynM;
  int* flags;                // [0] first diverged epoch (INT_MAX = none), [1] epoch (never reset)
  int base_epoch;            // epoch at the last reset (divergence step = epoch - base)
  cudaIpcMemHandle_t handle;
  void* opened[kMaxPeers];   // IPC mappings to close
  PeerBases bases;
  unsigned long long* post[kMaxPeers];  // &flag block of rank q ->flag[rank]
  int attached;              // ranks with a known base (own included)
  int fuse;
  cudaStream_t cap;
  cudaGraph_t graph[2];
  cudaGraphExec_t exec[2];   // [0] one step, [1] kGraphSteps steps
  double* graph_u;
};

namespace {

constexpr int kGraphSteps = 8;

bool fuse_ok(const Plan& p) { return p.kind == 0 && !p.tma_ok && p.own_idx == nullptr; }

int check_x(sdcsw_exchange* x, const char* where) {
  if (!x || !x->plan || !x->plan->alive) {
    set_error(std::string(where) + ": invalid exchange handle");
    return SDCSW_ERR_STATE;
  }
  return SDCSW_OK;
}

void drop_graphs(sdcsw_exchange* x) {
  for (int i = 0; i < 2; ++i) {
    if (x->exec[i]) cudaGraphExecDestroy(x->exec[i]);
    if (x->graph[i]) cudaGraphDestroy(x->graph[i]);
    x->exec[i] = nullptr;
    x->graph[i] = nullptr;
  }
  x->graph_u = nullptr;
}

// consumer of exchange k (1..K-1) of the current step
PeerWait peer_wait_args(const sdcsw_exchange* x, int k) {
  PeerWait pw{};
  pw.flags = x->pflag;
  pw.epoch = x->flags + 1;
  pw.k = k;
  pw.kx = x->K - 1;
  pw.world = x->world;
  pw.par_stride = (long long)x->M * 2 * (long long)x->S * 2;
  for (int q = 0; q < x->world; ++q) pw.post[q] = x->post[q];
  return pw;
}

// phase 0: f_E(u0) from the operand in xsyn1 (written by the previous step's
// closing solve or by the run's prep)
cudaError_t enqueue_phase(sdcsw_exchange* x, double2* u, int phase, cudaStream_t s) {
  const Plan& p = x->plan->p;
  const int M = x->M, K = x->K;
  const size_t S = x->S;
  const int cstride = M * (M + 4);
  const Work w = plan_work(p);
  cudaError_t e;
  if (phase == 0) return f_expl_prepped(p, w, x->xsyn1, x->fe0, 1, s, x->flags + 1, 0);
  if (phase < K) {
    const int k = phase;
    const bool first = k == 1;
    const PeerWait pw = peer_wait_args(x, k - 1);  // sweep k consumes exchange k - 1
    if (x->count == 0)
      return first ? cudaSuccess : launch_k(k_peer_post, dim3(1), dim3(32), 0, s, pw);
    {
      // first sweep: every node's tendencies are f(u0) (fe0, f_I(u0)); later:
      // the gathered [M][2][S] of the latest exchange (fe at 2j, fi at 2j + 1)
      const double2* fe = first ? x->fe0 : x->X;
      const double2* fi = first ? x->fe0 : x->X + S;
      const long long st = first ? 0 : 2;
      e = launch_sweep_nodes(p, M, x->lo, x->count, x->coef.data() + (size_t)(k - 1) * cstride, u,
                             fe, st, fi, st, first, nullptr, x->fi_loc, x->xsynM, s, 1, 0, 0, 0,
                             first ? nullptr : &pw);
      if (e != cudaSuccess) return e;
      if ((e = launch_synthesis(p, w, x->xsynM, x->count, s, nullptr)) != cudaSuccess) return e;
      if ((e = launch_ring(p, w, x->count, s)) != cudaSuccess) return e;
      if (x->fuse) {
        FuseArgs fz{};
        fz.mode = 4;
        fz.M = M;
        fz.phibar = p.phibar;
        fz.peer_world = x->world;
        fz.peer_lo = x->lo;
        fz.peer_epoch = x->flags + 1;
        fz.peer_k = k;
        fz.peer_kx = K - 1;
        fz.peer_fi = reinterpret_cast<const double*>(x->fi_loc);
        for (int q = 0; q < x->world; ++q) fz.peer_x[q] = x->bases.x[q];
        if ((e = launch_analysis_fused(p, w, x->count, fz, s)) != cudaSuccess) return e;
      } else {
        if ((e = launch_analysis(p, w, x->fe_loc, x->count, s)) != cudaSuccess) return e;
        dim3 grid((unsigned)((S + 255) / 256), x->count);
        e = launch_k(k_peer_publish, grid, 256, 0, s, (long long)S, M, x->lo,
                     (const double2*)x->fe_loc, (const double2*)x->fi_loc,
                     (const int*)(x->flags + 1), k, K - 1, x->bases, x->world);
        if (e != cudaSuccess) return e;
      }
    }
    return cudaSuccess;
  }
  // closing solve (K == 1: straight from f(u0))
  const bool first = K == 1;
  const double2* fe = first ? x->fe0 : x->X;
  const double2* fi = first ? x->fe0 : x->X + S;
  const long long st = first ? 0 : 2;
  const PeerWait pw = peer_wait_args(x, K - 1);
  return launch_final_node(p, M, x->coef.data() + (size_t)(K - 1) * cstride, u, fe, st, fi, st,
                           first, u, x->flags, x->flags + 1, x->xsyn1, s, 1, 0, 0,
                           first ? nullptr : &pw);
}

cudaError_t enqueue_step(sdcsw_exchange* x, double2* u, cudaStream_t s) {
  for (int ph = 0; ph <= x->K; ++ph) {
    cudaError_t e = enqueue_phase(x, u, ph, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int ready(sdcsw_exchange* x, const char* where) {
  if (x->attached != x->world) {
    set_error(std::string(where) + ": peers not attached (open_peers / attach_peer)");
    return SDCSW_ERR_STATE;
  }
  return SDCSW_OK;
}

}  // namespace

extern "C" {

int sdcsw_exchange_create(sdcsw_plan* h, int n_nodes, int n_sweeps, const double* coef,
                          int n_coef, int world, int rank, sdcsw_exchange** out) {
  if (!h || !h->alive) {
    set_error("sdcsw_exchange_create: invalid plan handle");
    return SDCSW_ERR_STATE;
  }
  const Plan& p = h->p;
  const int M = n_nodes, K = n_sweeps;
  if (!out || !coef || M < 1 || M > 16 || K < 1 || world < 1 || world > kMaxPeers || rank < 0 ||
      rank >= world) {
    set_error("sdcsw_exchange_create: bad node / sweep / rank count");
    return SDCSW_ERR_PARAM;
  }
  if (p.kind != 0 || p.split_S > 1) {
    set_error("sdcsw_exchange_create: unsplit spherical plans only");
    return SDCSW_ERR_STATE;
  }
  const int need = (K - 1) * M * (M + 4) + (M + 4);
  if (n_coef < need) {
    set_error("sdcsw_exchange_create: coefficient array too short");
    return SDCSW_ERR_PARAM;
  }
  const int per = (M + world - 1) / world;
  const int lo = rank * per < M ? rank * per : M;
  const int count = M - lo < per ? M - lo : per;
  if (count > p.max_batch) {
    set_error("sdcsw_exchange_create: plan max_batch < nodes per rank");
    return SDCSW_ERR_PARAM;
  }
  sdcsw_exchange* x = new (std::nothrow) sdcsw_exchange();
  if (!x) return SDCSW_ERR_PARAM;
  x->plan = h;
  x->M = M;
  x->K = K;
  x->world = world;
  x->rank = rank;
  x->lo = lo;
  x->count = count;
  x->coef.assign((size_t)K * M * (M + 4), 0.0);
  std::memcpy(x->coef.data(), coef, (size_t)(K - 1) * M * (M + 4) * sizeof(double));
  std::memcpy(x->coef.data() + (size_t)(K - 1) * M * (M + 4),
              coef + (size_t)(K - 1) * M * (M + 4), (size_t)(M + 4) * sizeof(double));
  x->S = (size_t)3 * p.C;
  x->fuse = fuse_ok(p) ? 1 : 0;
  const size_t xbytes = (size_t)2 * M * 2 * x->S * sizeof(double2);
  const size_t cnt = count > 0 ? count : 1;
  const size_t xs = (size_t)p.rows * kXsyn * sizeof(double);
  const size_t lbytes = (1 + 2 * cnt) * x->S * sizeof(double2) + xs * (1 + cnt) + 2 * sizeof(int);
  cudaError_t e = cudaSetDevice(p.device);
  if (e == cudaSuccess) e = cudaMalloc(&x->mem, xbytes + sizeof(PeerFlags));
  if (e == cudaSuccess) e = cudaMalloc(&x->local, lbytes);
  if (e == cudaSuccess) e = cudaMemset(x->mem, 0, xbytes + sizeof(PeerFlags));
  if (e == cudaSuccess) e = cudaMemset(x->local, 0, lbytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&x->handle, x->mem);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&x->cap, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any peer can post
  if (e != cudaSuccess) {
    if (x->mem) cudaFree(x->mem);
    if (x->local) cudaFree(x->local);
    delete x;
    return cuda_status(e, "sdcsw_exchange_create");
  }
  x->X = reinterpret_cast<double2*>(x->mem);
  x->pflag = reinterpret_cast<PeerFlags*>(x->mem + xbytes);
  double2* q = reinterpret_cast<double2*>(x->local);
  x->fe0 = q; q += x->S;
  x->fe_loc = q; q += cnt * x->S;
  x->fi_loc = q; q += cnt * x->S;
  x->xsyn1 = reinterpret_cast<double*>(q);
  x->xsynM = x->xsyn1 + (size_t)p.rows * kXsyn;
  x->flags = reinterpret_cast<int*>(x->xsynM + (size_t)p.rows * kXsyn * cnt);
  const int init[2] = {INT_MAX, 0};
  cudaMemcpy(x->flags, init, sizeof(init), cudaMemcpyHostToDevice);
  x->bases.x[rank] = reinterpret_cast<double*>(x->X);
  x->post[rank] = &x->pflag->flag[rank];
  x->attached = 1;
  *out = x;
  return SDCSW_OK;
}

int sdcsw_exchange_ipc_handle(sdcsw_exchange* x, void* handle, int bytes) {
  if (int st = check_x(x, "sdcsw_exchange_ipc_handle")) return st;
  if (!handle || bytes < (int)sizeof(cudaIpcMemHandle_t)) return SDCSW_ERR_PARAM;
  std::memcpy(handle, &x->handle, sizeof(cudaIpcMemHandle_t));
  return SDCSW_OK;
}

static int attach(sdcsw_exchange* x, int q, char* base) {
  const size_t xbytes = (size_t)2 * x->M * 2 * x->S * sizeof(double2);
  const bool fresh = q != x->rank && x->bases.x[q] == nullptr;
  x->bases.x[q] = reinterpret_cast<double*>(base);
  // this rank posts into flag[rank] of rank q's flag block
  x->post[q] = &reinterpret_cast<PeerFlags*>(base + xbytes)->flag[x->rank];
  if (fresh) ++x->attached;
  drop_graphs(x);
  return SDCSW_OK;
}

int sdcsw_exchange_open_peers(sdcsw_exchange* x, const void* handles, int bytes_each) {
  if (int st = check_x(x, "sdcsw_exchange_open_peers")) return st;
  if (!handles || bytes_each < (int)sizeof(cudaIpcMemHandle_t)) return SDCSW_ERR_PARAM;
  cudaError_t e = cudaSetDevice(x->plan->p.device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  for (int q = 0; q < x->world; ++q) {
    if (q == x->rank || x->opened[q]) continue;
    cudaIpcMemHandle_t hq;
    std::memcpy(&hq, static_cast<const char*>(handles) + (size_t)q * bytes_each, sizeof(hq));
    void* ptr = nullptr;
    e = cudaIpcOpenMemHandle(&ptr, hq, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcOpenMemHandle");
    x->opened[q] = ptr;
    attach(x, q, static_cast<char*>(ptr));
  }
  return SDCSW_OK;
}

int sdcsw_exchange_base(sdcsw_exchange* x, void** base) {
  if (int st = check_x(x, "sdcsw_exchange_base")) return st;
  if (!base) return SDCSW_ERR_PARAM;
  *base = x->mem;
  return SDCSW_OK;
}

int sdcsw_exchange_attach_peer(sdcsw_exchange* x, int peer, void* base) {
  if (int st = check_x(x, "sdcsw_exchange_attach_peer")) return st;
  if (peer < 0 || peer >= x->world || peer == x->rank || !base) return SDCSW_ERR_PARAM;
  return attach(x, peer, static_cast<char*>(base));
}

int sdcsw_exchange_phase(sdcsw_exchange* x, double* u, int phase, void* stream) {
  if (int st = check_x(x, "sdcsw_exchange_phase")) return st;
  if (int st = ready(x, "sdcsw_exchange_phase")) return st;
  if (!u || phase < 0 || phase > x->K) return SDCSW_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(x->plan->p.device);
  if (e == cudaSuccess && phase == 0)
    e = launch_synth_prep(x->plan->p, (const double2*)u, 1, x->xsyn1, s);
  if (e == cudaSuccess) e = enqueue_phase(x, (double2*)u, phase, s);
  return cuda_status(e, "sdcsw_exchange_phase");
}

int sdcsw_exchange_post(sdcsw_exchange* x, int k, void* stream) {
  if (int st = check_x(x, "sdcsw_exchange_post")) return st;
  if (int st = ready(x, "sdcsw_exchange_post")) return st;
  if (k < 1 || k >= x->K) return SDCSW_ERR_PARAM;
  cudaError_t e = cudaSetDevice(x->plan->p.device);
  if (e == cudaSuccess)
    e = launch_k(k_peer_post, dim3(1), dim3(32), 0, (cudaStream_t)stream, peer_wait_args(x, k));
  return cuda_status(e, "sdcsw_exchange_post");
}

int sdcsw_exchange_run(sdcsw_exchange* x, double* u, int n_steps, int use_graph, void* stream) {
  if (int st = check_x(x, "sdcsw_exchange_run")) return st;
  if (int st = ready(x, "sdcsw_exchange_run")) return st;
  if (!u || n_steps < 0) return SDCSW_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(x->plan->p.device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  if (n_steps == 0) return SDCSW_OK;
  // the caller may have changed u: rebuild its synthesis operand
  e = launch_synth_prep(x->plan->p, (const double2*)u, 1, x->xsyn1, s);
  if (e != cudaSuccess) return cuda_status(e, "sdcsw_exchange_run prep");
  if (!use_graph) {
    for (int i = 0; i < n_steps; ++i)
      if ((e = enqueue_step(x, (double2*)u, s)) != cudaSuccess)
        return cuda_status(e, "sdcsw_exchange_run");
    return SDCSW_OK;
  }
  if (!x->exec[0] || x->graph_u != u) {
    drop_graphs(x);
    const int steps[2] = {1, kGraphSteps};
    for (int g = 0; g < 2; ++g) {
      e = cudaStreamBeginCapture(x->cap, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamBeginCapture");
      cudaError_t le = cudaSuccess;
      for (int i = 0; i < steps[g] && le == cudaSuccess; ++i)
        le = enqueue_step(x, (double2*)u, x->cap);
      e = cudaStreamEndCapture(x->cap, &x->graph[g]);
      if (le != cudaSuccess) return cuda_status(le, "capture step");
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamEndCapture");
      if ((e = cudaGraphInstantiate(&x->exec[g], x->graph[g], 0)) != cudaSuccess)
        return cuda_status(e, "cudaGraphInstantiate");
    }
    x->graph_u = u;
  }
  int i = 0;
  for (; i + kGraphSteps <= n_steps; i += kGraphSteps)
    if ((e = cudaGraphLaunch(x->exec[1], s)) != cudaSuccess) return cuda_status(e, "cudaGraphLaunch");
  for (; i < n_steps; ++i)
    if ((e = cudaGraphLaunch(x->exec[0], s)) != cudaSuccess) return cuda_status(e, "cudaGraphLaunch");
  return SDCSW_OK;
}

int sdcsw_exchange_set_option(sdcsw_exchange* x, int option, int value) {
  if (int st = check_x(x, "sdcsw_exchange_set_option")) return st;
  if (option != 0) return SDCSW_ERR_PARAM;
  if (value && !fuse_ok(x->plan->p)) {
    set_error("sdcsw_exchange_set_option: the plan's analysis has no fused epilogue");
    return SDCSW_ERR_PARAM;
  }
  x->fuse = value ? 1 : 0;
  drop_graphs(x);
  return SDCSW_OK;
}

int sdcsw_exchange_info(sdcsw_exchange* x, int* node_lo, int* node_count, int* launches) {
  if (int st = check_x(x, "sdcsw_exchange_info")) return st;
  if (node_lo) *node_lo = x->lo;
  if (node_count) *node_count = x->count;
  if (launches) {
    // init f_E (3) + per full sweep (node, synthesis, ring, analysis [+ copy];
    // no nodes: a post from sweep 2 on) + closing solve
    *launches = 3 + 1 + (x->count > 0 ? (x->K - 1) * (x->fuse ? 4 : 5) : (x->K > 2 ? x->K - 2 : 0));
  }
  return SDCSW_OK;
}

int sdcsw_exchange_diverged(sdcsw_exchange* x, int* step_index) {
  if (int st = check_x(x, "sdcsw_exchange_diverged")) return st;
  if (!step_index) return SDCSW_ERR_PARAM;
  int v[2];
  cudaSetDevice(x->plan->p.device);
  cudaDeviceSynchronize();
  cudaError_t e = cudaMemcpy(v, x->flags, sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "sdcsw_exchange_diverged");
  *step_index = v[0] == INT_MAX ? 0 : v[0] - x->base_epoch;
  return SDCSW_OK;
}

int sdcsw_exchange_reset(sdcsw_exchange* x, void* stream) {
  if (int st = check_x(x, "sdcsw_exchange_reset")) return st;
  // the epoch is never reset (exchange numbers stay in lock step across
  // ranks): divergence is reported relative to the epoch at the reset
  cudaStream_t s = (cudaStream_t)stream;
  int epoch = 0;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaMemcpy(&epoch, x->flags + 1, sizeof(int), cudaMemcpyDeviceToHost);
  const int none = INT_MAX;
  if (e == cudaSuccess) e = cudaMemcpyAsync(x->flags, &none, sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  x->base_epoch = epoch;
  return cuda_status(e, "sdcsw_exchange_reset");
}

int sdcsw_exchange_destroy(sdcsw_exchange* x) {
  if (!x) return SDCSW_ERR_STATE;
  cudaSetDevice(x->plan->p.device);
  cudaDeviceSynchronize();
  drop_graphs(x);
  for (int q = 0; q < kMaxPeers; ++q)
    if (x->opened[q]) cudaIpcCloseMemHandle(x->opened[q]);
  cudaStreamDestroy(x->cap);
  cudaFree(x->mem);
  cudaFree(x->local);
  delete x;
  return SDCSW_OK;
}

}  // extern "C"
