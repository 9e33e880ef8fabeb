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
//
// With S > 1 spectral parts (more GPUs than nodes) the world is G
// node groups x S parts (rank = g S + sp): part sp owns the wavenumber pairs
// (m, T - m) dealt to it, the state is m-partitioned, and every f_E also
// exchanges the synthesised Fourier coefficients inside the node group's
// spectral group - the split synthesis stores its part straight into every
// spectral peer's buffer and the ring kernel posts / waits (SynDst, RingPeer).
// The node exchange then runs among the G ranks that share part sp.
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
    if (pw.world > 1) __threadfence_system();
    for (int q = 0; q < pw.world; ++q) atomicMax_system(pw.post[q], n);
  }
}

// Post only, Fourier channel: exchange fseq + 1 (for single-stream drivers)
__global__ void k_fourier_post(RingPeer rp) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  if (threadIdx.x == 0) {
    const unsigned long long n = *rp.fseq + 1;
    if (rp.world > 1) __threadfence_system();
    for (int q = 0; q < rp.world; ++q) atomicMax_system(rp.post[q], n);
  }
}

}  // namespace sdcsw

using namespace sdcsw;

struct sdcsw_exchange {
  sdcsw_plan* plan;
  int M, K;
  int world, rank;           // all ranks
  int S, sp, G, g;           // spectral parts, own part, node groups, own node group
  int lo, count, per;        // own node block (per = ceil(M / G))
  std::vector<double> coef;  // K blocks of M (M + 4); block K-1 = final (M + 4)
  size_t S1;                 // one state, in double2
  size_t xbytes, fbytes;     // exchange buffer X, Fourier buffer F (both parities)
  long long fpar;            // double2 per parity of F
  long long fpart;           // double2 per part of F at batch 1 (J Lp 8)
  char* mem;                 // IPC allocation: X | F | node flags | Fourier flags
  double2* X;                // [2][M][2][S1]
  double2* F;                // [2][S][max_batch][J][Lp][4][2] (S > 1)
  PeerFlags *nflag, *fflag;
  char* local;               // private buffers
  double2 *fe0, *fe_loc, *fi_loc;
  double *xsyn1, *xsynM;
  int* flags;                // [0] first diverged epoch (INT_MAX = none), [1] epoch (never reset),
                             // [2..4] wait timeout: peer + 1 (0 = none), channel, exchange number
  unsigned long long timeout_ns;  // bound of every device wait on a peer's post (option 1)
  unsigned long long* fseq;  // completed Fourier exchanges
  unsigned int* done;        // ring CTA counter
  int base_epoch;            // epoch at the last reset (divergence step = epoch - base)
  cudaIpcMemHandle_t handle;
  void* opened[kMaxPeers];   // IPC mappings to close
  char* base[kMaxPeers];     // every rank's allocation (own included)
  int attached;              // ranks with a known base (own included)
  int fuse;
  cudaStream_t cap;
  cudaGraph_t graph[2];
  cudaGraphExec_t exec[2];   // [0] one step, [1] kGraphSteps steps
  double* graph_u;
};

namespace {

constexpr int kGraphSteps = 8;

bool fuse_ok(const Plan& p) { return p.kind == 0 && !p.tma_ok; }

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

PeerFlags* nflag_of(const sdcsw_exchange* x, int r) {
  return reinterpret_cast<PeerFlags*>(x->base[r] + x->xbytes + x->fbytes);
}
PeerFlags* fflag_of(const sdcsw_exchange* x, int r) { return nflag_of(x, r) + 1; }

// consumer of node exchange k (1..K-1) of the current step; peers = the G
// ranks sharing part sp (node group i -> rank i S + sp)
PeerWait peer_wait_args(const sdcsw_exchange* x, int k) {
  PeerWait pw{};
  pw.flags = x->nflag;
  pw.epoch = x->flags + 1;
  pw.k = k;
  pw.kx = x->K - 1;
  pw.world = x->G;
  pw.par_stride = (long long)x->M * 2 * (long long)x->S1 * 2;
  for (int i = 0; i < x->G; ++i) pw.post[i] = &nflag_of(x, i * x->S + x->sp)->flag[x->g];
  pw.to = PeerTimeout{x->flags + 2, x->timeout_ns};
  return pw;
}

// Fourier channel: peers = the S parts of node group g (rank g S + q)
RingPeer ring_peer_args(const sdcsw_exchange* x) {
  RingPeer rp{};
  rp.flags = x->fflag;
  rp.fseq = x->fseq;
  rp.done = x->done;
  rp.world = x->S;
  rp.par_stride = x->fpar;
  for (int q = 0; q < x->S; ++q) rp.post[q] = &fflag_of(x, x->g * x->S + q)->flag[x->sp];
  rp.to = PeerTimeout{x->flags + 2, x->timeout_ns};
  return rp;
}

SynDst syn_dst_args(const sdcsw_exchange* x, int nb) {
  SynDst d{};
  d.n = x->S;
  d.par_stride = x->fpar;
  d.fseq = x->fseq;
  for (int q = 0; q < x->S; ++q)
    d.dst[q] = reinterpret_cast<double2*>(x->base[x->g * x->S + q] + x->xbytes) +
               (size_t)x->sp * nb * x->fpart;
  return d;
}

// f_E, first half: synthesis of the operand xs (nb states); split: into every
// spectral peer's Fourier buffer
cudaError_t f_first(sdcsw_exchange* x, const double* xs, int nb, int* counter, cudaStream_t s) {
  const Plan& p = x->plan->p;
  if (x->S > 1) {
    return launch_synthesis_peer(p, xs, nb, s, syn_dst_args(x, nb), counter);
  }
  return launch_synthesis(p, plan_work(p), xs, nb, s, counter);
}

// f_E, second half: ring (split: after every part arrived)
cudaError_t f_ring(sdcsw_exchange* x, int nb, cudaStream_t s) {
  const Plan& p = x->plan->p;
  if (x->S > 1) return launch_ring_peer(p, plan_work(p), x->F, nb, s, ring_peer_args(x));
  return launch_ring(p, plan_work(p), nb, s);
}

// Half-phases of a step: h = 2k and 2k + 1 for f_E k = 0..K-1 (k = 0: f_E(u0)
// from the operand in xsyn1, written by the previous step's closing solve or
// the run's prep; k >= 1: full sweep k, publishing node exchange k), h = 2K:
// the closing solve.  2k: [node kernel k] + synthesis; 2k + 1: ring + analysis.
cudaError_t enqueue_half(sdcsw_exchange* x, double2* u, int h, cudaStream_t s) {
  const Plan& p = x->plan->p;
  const int M = x->M, K = x->K;
  const size_t S1 = x->S1;
  const int cstride = M * (M + 4);
  const Work w = plan_work(p);
  cudaError_t e;
  if (h == 2 * K) {  // closing solve (K == 1: straight from f(u0))
    const bool first = K == 1;
    const double2* fe = first ? x->fe0 : x->X;
    const double2* fi = first ? x->fe0 : x->X + S1;
    const long long st = first ? 0 : 2;
    const PeerWait pw = peer_wait_args(x, K - 1);
    return launch_final_node(p, M, x->coef.data() + (size_t)(K - 1) * cstride, u, fe, st, fi, st,
                             first, u, x->flags, x->flags + 1, x->xsyn1, s, 1, 0, 0,
                             first ? nullptr : &pw);
  }
  const int k = h / 2;
  if (k == 0) {
    if (h == 0) return f_first(x, x->xsyn1, 1, x->flags + 1, s);
    if ((e = f_ring(x, 1, s)) != cudaSuccess) return e;
    return launch_analysis(p, w, x->fe0, 1, s);
  }
  const bool first = k == 1;
  const PeerWait pw = peer_wait_args(x, k - 1);  // sweep k consumes node exchange k - 1
  if (x->count == 0) {
    if (h % 2 == 0 && !first) return launch_k(k_peer_post, dim3(1), dim3(32), 0, s, pw);
    return cudaSuccess;
  }
  if (h % 2 == 0) {
    // first sweep: every node's tendencies are f(u0) (fe0, f_I(u0)); later:
    // the gathered [M][2][S1] of the latest exchange (fe at 2j, fi at 2j + 1)
    const double2* fe = first ? x->fe0 : x->X;
    const double2* fi = first ? x->fe0 : x->X + S1;
    const long long st = first ? 0 : 2;
    e = launch_sweep_nodes(p, M, x->lo, x->count, x->coef.data() + (size_t)(k - 1) * cstride, u,
                           fe, st, fi, st, first, nullptr, x->fi_loc, x->xsynM, s, 1, 0, 0, 0,
                           first ? nullptr : &pw);
    if (e != cudaSuccess) return e;
    return f_first(x, x->xsynM, x->count, nullptr, s);
  }
  if ((e = f_ring(x, x->count, s)) != cudaSuccess) return e;
  if (x->fuse) {
    FuseArgs fz{};
    fz.mode = 4;
    fz.M = M;
    fz.phibar = p.phibar;
    fz.peer_world = x->G;
    fz.peer_lo = x->lo;
    fz.peer_epoch = x->flags + 1;
    fz.peer_k = k;
    fz.peer_kx = K - 1;
    fz.peer_fi = reinterpret_cast<const double*>(x->fi_loc);
    for (int i = 0; i < x->G; ++i)
      fz.peer_x[i] = reinterpret_cast<double*>(x->base[i * x->S + x->sp]);
    return launch_analysis_fused(p, w, x->count, fz, s);
  }
  if ((e = launch_analysis(p, w, x->fe_loc, x->count, s)) != cudaSuccess) return e;
  PeerBases pb{};
  for (int i = 0; i < x->G; ++i) pb.x[i] = reinterpret_cast<double*>(x->base[i * x->S + x->sp]);
  dim3 grid((unsigned)((S1 + 255) / 256), x->count);
  return launch_k(k_peer_publish, grid, 256, 0, s, (long long)S1, M, x->lo,
                  (const double2*)x->fe_loc, (const double2*)x->fi_loc,
                  (const int*)(x->flags + 1), k, K - 1, pb, x->G);
}

cudaError_t enqueue_step(sdcsw_exchange* x, double2* u, cudaStream_t s) {
  for (int h = 0; h <= 2 * x->K; ++h) {
    cudaError_t e = enqueue_half(x, u, h, s);
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
  return sdcsw_exchange_create_split(h, n_nodes, n_sweeps, coef, n_coef, world, rank, 1, out);
}

int sdcsw_exchange_create_split(sdcsw_plan* h, int n_nodes, int n_sweeps, const double* coef,
                                int n_coef, int world, int rank, int spectral_parts,
                                sdcsw_exchange** out) {
  if (!h || !h->alive) {
    set_error("sdcsw_exchange_create: invalid plan handle");
    return SDCSW_ERR_STATE;
  }
  Plan& p = h->p;
  const int M = n_nodes, K = n_sweeps, S = spectral_parts;
  if (!out || !coef || M < 1 || M > 16 || K < 1 || world < 1 || world > kMaxPeers || rank < 0 ||
      rank >= world || S < 1 || world % S || S > p.L) {
    set_error("sdcsw_exchange_create: bad node / sweep / rank / part count");
    return SDCSW_ERR_PARAM;
  }
  const int G = world / S;
  if (S > 1 && G > M) {
    set_error("sdcsw_exchange_create: with spectral parts every node group needs a node");
    return SDCSW_ERR_PARAM;
  }
  if (p.kind != 0 || p.split_S > 1) {
    set_error("sdcsw_exchange_create: unsplit spherical plans only (the exchange splits it)");
    return SDCSW_ERR_STATE;
  }
  const int need = (K - 1) * M * (M + 4) + (M + 4);
  if (n_coef < need) {
    set_error("sdcsw_exchange_create: coefficient array too short");
    return SDCSW_ERR_PARAM;
  }
  const int g = rank / S, sp = rank % S;
  const int per = (M + G - 1) / G;
  const int lo = g * per < M ? g * per : M;
  const int count = M - lo < per ? M - lo : per;
  if (count > p.max_batch) {
    set_error("sdcsw_exchange_create: plan max_batch < nodes per rank");
    return SDCSW_ERR_PARAM;
  }
  // the Fourier exchange buffer follows the split's part-major layout
  int Lp = p.L;
  if (S > 1) {
    std::vector<int> part(p.L), cnt(S, 0);
    for (int i = 0, m = 0; m <= p.T - m; ++m, ++i) part[m] = part[p.T - m] = i % S;
    for (int m = 0; m < p.L; ++m) ++cnt[part[m]];
    Lp = 0;
    for (int q = 0; q < S; ++q) Lp = cnt[q] > Lp ? cnt[q] : Lp;
  }
  sdcsw_exchange* x = new (std::nothrow) sdcsw_exchange();
  if (!x) return SDCSW_ERR_PARAM;
  x->plan = h;
  x->M = M;
  x->K = K;
  x->world = world;
  x->rank = rank;
  x->S = S;
  x->sp = sp;
  x->G = G;
  x->g = g;
  x->lo = lo;
  x->count = count;
  x->per = per;
  x->coef.assign((size_t)K * M * (M + 4), 0.0);
  std::memcpy(x->coef.data(), coef, (size_t)(K - 1) * M * (M + 4) * sizeof(double));
  std::memcpy(x->coef.data() + (size_t)(K - 1) * M * (M + 4),
              coef + (size_t)(K - 1) * M * (M + 4), (size_t)(M + 4) * sizeof(double));
  x->S1 = (size_t)3 * p.C;
  x->fuse = fuse_ok(p) ? 1 : 0;
  x->xbytes = (size_t)2 * M * 2 * x->S1 * sizeof(double2);
  x->fpart = (long long)p.J * Lp * 8;
  x->fpar = S > 1 ? (long long)S * p.max_batch * x->fpart : 0;
  x->fbytes = (size_t)2 * x->fpar * sizeof(double2);
  const size_t mbytes = x->xbytes + x->fbytes + 2 * sizeof(PeerFlags);
  const size_t cnt = count > 0 ? count : 1;
  const size_t xs = (size_t)p.rows * kXsyn * sizeof(double);
  const size_t lbytes = (1 + 2 * cnt) * x->S1 * sizeof(double2) + xs * (1 + cnt) + 64;
  cudaError_t e = cudaSetDevice(p.device);
  if (e == cudaSuccess) e = cudaMalloc(&x->mem, mbytes);
  if (e == cudaSuccess) e = cudaMalloc(&x->local, lbytes);
  if (e == cudaSuccess) e = cudaMemset(x->mem, 0, mbytes);
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
  x->F = reinterpret_cast<double2*>(x->mem + x->xbytes);
  x->nflag = reinterpret_cast<PeerFlags*>(x->mem + x->xbytes + x->fbytes);
  x->fflag = x->nflag + 1;
  double2* q = reinterpret_cast<double2*>(x->local);
  x->fe0 = q; q += x->S1;
  x->fe_loc = q; q += cnt * x->S1;
  x->fi_loc = q; q += cnt * x->S1;
  x->xsyn1 = reinterpret_cast<double*>(q);
  x->xsynM = x->xsyn1 + (size_t)p.rows * kXsyn;
  char* tail = reinterpret_cast<char*>(x->xsynM + (size_t)p.rows * kXsyn * cnt);
  x->fseq = reinterpret_cast<unsigned long long*>(tail);
  x->done = reinterpret_cast<unsigned int*>(tail + 8);
  x->flags = reinterpret_cast<int*>(tail + 16);
  const int init[5] = {INT_MAX, 0, 0, 0, 0};
  cudaMemcpy(x->flags, init, sizeof(init), cudaMemcpyHostToDevice);
  x->timeout_ns = 30ull * 1000000000ull;
  x->base[rank] = x->mem;
  x->attached = 1;
  if (S > 1) {  // the plan keeps own wavenumbers only; its Fourier buffer is F
    const int st = sdcsw_plan_set_split(h, S, sp, x->F, (long long)(x->fpar * sizeof(double2)));
    if (st != SDCSW_OK) {
      cudaFree(x->mem);
      cudaFree(x->local);
      cudaStreamDestroy(x->cap);
      delete x;
      return st;
    }
  }
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
  if (q != x->rank && x->base[q] == nullptr) ++x->attached;
  x->base[q] = base;
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
  if (!u || phase < 0 || phase > 2 * x->K) return SDCSW_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(x->plan->p.device);
  if (e == cudaSuccess && phase == 0)
    e = launch_synth_prep(x->plan->p, (const double2*)u, 1, x->xsyn1, s);
  if (e == cudaSuccess) e = enqueue_half(x, (double2*)u, phase, s);
  return cuda_status(e, "sdcsw_exchange_phase");
}

int sdcsw_exchange_post(sdcsw_exchange* x, int channel, int k, void* stream) {
  if (int st = check_x(x, "sdcsw_exchange_post")) return st;
  if (int st = ready(x, "sdcsw_exchange_post")) return st;
  cudaError_t e = cudaSetDevice(x->plan->p.device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  cudaStream_t s = (cudaStream_t)stream;
  if (channel == 0) {
    if (k < 1 || k >= x->K) return SDCSW_ERR_PARAM;
    e = launch_k(k_peer_post, dim3(1), dim3(32), 0, s, peer_wait_args(x, k));
  } else if (channel == 1) {
    if (x->S < 2) return SDCSW_ERR_PARAM;
    e = launch_k(k_fourier_post, dim3(1), dim3(32), 0, s, ring_peer_args(x));
  } else {
    return SDCSW_ERR_PARAM;
  }
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
    for (int gi = 0; gi < 2; ++gi) {
      e = cudaStreamBeginCapture(x->cap, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamBeginCapture");
      cudaError_t le = cudaSuccess;
      for (int i = 0; i < steps[gi] && le == cudaSuccess; ++i)
        le = enqueue_step(x, (double2*)u, x->cap);
      e = cudaStreamEndCapture(x->cap, &x->graph[gi]);
      if (le != cudaSuccess) return cuda_status(le, "capture step");
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamEndCapture");
      if ((e = cudaGraphInstantiate(&x->exec[gi], x->graph[gi], 0)) != cudaSuccess)
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
  if (option == 1) {  // bound of every device wait on a peer, milliseconds
    if (value < 1) {
      set_error("sdcsw_exchange_set_option: the wait bound must be >= 1 ms");
      return SDCSW_ERR_PARAM;
    }
    x->timeout_ns = (unsigned long long)value * 1000000ull;
    drop_graphs(x);  // the bound is a kernel argument captured in the graphs
    return SDCSW_OK;
  }
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
  int v[5];
  cudaSetDevice(x->plan->p.device);
  cudaDeviceSynchronize();
  cudaError_t e = cudaMemcpy(v, x->flags, sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "sdcsw_exchange_diverged");
  *step_index = v[0] == INT_MAX ? 0 : v[0] - x->base_epoch;
  if (v[2] != 0) {
    const int peer = v[2] - 1;
    const int rank = v[3] == 0 ? peer * x->S + x->sp : x->g * x->S + peer;
    set_error("sdcsw_exchange: rank " + std::to_string(rank) + " did not post " +
              (v[3] == 0 ? "node" : "Fourier") + " exchange " + std::to_string(v[4]) + " within " +
              std::to_string(x->timeout_ns / 1000000ull) +
              " ms (peer died or stopped stepping); the state is invalid");
    return SDCSW_ERR_PEER;
  }
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
  const int none = INT_MAX, clear[3] = {0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(x->flags, &none, sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(x->flags + 2, clear, sizeof(clear), cudaMemcpyHostToDevice, s);
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
