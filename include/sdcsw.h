/*
 * sdcsw.h - C ABI of libsdcsw.so, the B200 (sm_100a) hot path of parallel
 * spectral deferred corrections (dSDC, MIN-SR-FLEX, IMEX) applied to rotating
 * shallow water on the sphere in a spherical-harmonic discretisation.
 *
 * Plain C types only: device buffers are raw pointers the caller owns
 * (e.g. torch.Tensor.data_ptr()), streams are cudaStream_t passed as void*.
 * Every entry point returns an sdcsw_status and never throws; the message of
 * the last failure on the calling thread is sdcsw_last_error().
 *
 * State layout (fixed): complex128 interleaved (re, im); one state is three
 * fields (Phi', zeta, delta) of C = (T+1)(T+2)/2 coefficients each, triangular
 * m-major: idx(m, n) = m (T+1) - m (m-1)/2 + (n - m).  A batch of nb states is
 * nb consecutive states (stride 3 C complex).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the parsdc reference package, pkg/src/parsdc/).
 */
#ifndef SDCSW_H
#define SDCSW_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SDCSW_OK = 0,
  SDCSW_ERR_PARAM = 1,    /* -> ParameterError (errors.py:4) */
  SDCSW_ERR_CUDA = 2,     /* launch / allocation failure -> DeviceError */
  SDCSW_ERR_STATE = 3,    /* call on a destroyed or mismatched handle */
  SDCSW_ERR_DIVERGED = 4, /* non-finite state -> DivergenceError (integrators.py:544-548) */
  SDCSW_ERR_PEER = 5      /* a peer did not post an exchange within the wait bound -> DeviceError */
} sdcsw_status;

typedef struct sdcsw_plan sdcsw_plan;
typedef struct sdcsw_stepper sdcsw_stepper;

typedef struct {
  int trunc;      /* spectral truncation T */
  int nlat;       /* Gaussian latitudes (even) */
  int nlon;       /* longitudes, 2^k or 3*2^k, >= 2T+2 */
  int max_batch;  /* largest nb any call on this plan will use */
  double radius;  /* a */
  double omega;   /* rotation rate */
  double phibar;  /* mean geopotential g*H */
} sdcsw_config;

/* Host-built constants uploaded once; the plan owns the device copies and the
 * transform workspaces.  Tables are parity-sorted, padded rows:
 * ptab/htab [rows][nlat/2], rowoff [T+2], n_even [T+1] (padded even-row count
 * per m), row_n [rows] (degree n of each row, -1 = padding), lam [C]
 * (n(n+1)/a^2), mu_north/w_north [nlat/2] (northern Gaussian nodes/weights,
 * pole first).  Replaces the problem construction of the planar template
 * (problems/swe.py:77-138) for the spherical problem the reference scopes out. */
int sdcsw_plan_create(int device, const sdcsw_config* cfg, const double* mu_north,
                      const double* w_north, const double* ptab, const double* htab,
                      const int* rowoff, const int* n_even, const int* row_n,
                      const double* lam, sdcsw_plan** out);
int sdcsw_plan_destroy(sdcsw_plan* plan);

typedef struct {
  int n_grid;                /* N: 8, 12, 16, 24, ..., 768, 1024 (2^k or 3*2^k) */
  int max_batch;             /* largest nb any call on this plan will use */
  double domain_length;      /* L (informational; the wavenumbers carry it) */
  double mean_geopotential;  /* phibar > 0 */
  double coriolis;           /* f0 */
  double hyperviscosity;     /* nu >= 0 */
} sdcsw_planar_config;

/* Planar doubly periodic problem (PlanarShallowWater, problems/swe.py:57-138):
 * state = three [N][N/2+1] rfft2 spectra (Phi', zeta, delta), C = N (N/2+1)
 * coefficients per field.  kx [N] = 2 pi fftfreq, ky [N/2+1] = 2 pi rfftfreq,
 * lam [C] = kx^2 + ky^2 (the reference's laplacian_symbol), host arrays built
 * with the reference's expressions.  sdcsw_f_expl / f_impl / implicit_solve /
 * sweep_nodes / final_node / the steppers accept the plan; the spherical-only
 * entry points (transform stages, workspaces, spectral split) reject it. */
int sdcsw_plan_create_planar(int device, const sdcsw_planar_config* cfg, const double* kx,
                             const double* ky, const double* lam, sdcsw_plan** out);

/* fe[b] = f_E(u[b]) for b < nb.  Replaces SplitProblem.f_expl (core.py:102-104)
 * and the planar _f_expl (problems/swe.py:174-196). */
int sdcsw_f_expl(sdcsw_plan* plan, const double* u, double* fe, int nb, void* stream);

/* fi[b] = f_I(u[b]) = (-phibar delta, 0, lam Phi').  Replaces
 * SplitProblem.f_impl (core.py:106-108) / problems/swe.py:157-163. */
int sdcsw_f_impl(sdcsw_plan* plan, const double* u, double* fi, int nb, void* stream);

/* u[b] solves u - alpha_b f_I(u) = beta[b]; coef is HOST memory [nb][3] =
 * (alpha, alpha*phibar, alpha*alpha*phibar).  alpha == 0 copies beta.
 * Replaces SplitProblem.implicit_solve (core.py:110-114) /
 * problems/swe.py:165-172. */
int sdcsw_implicit_solve(sdcsw_plan* plan, const double* coef, const double* beta, double* u,
                         int nb, void* stream);

/* Phase one + solve of one diagonal sweep for nodes [node_lo, node_lo+count):
 *   F_j = fe_j + fi_j;  beta_m = u0 + sum_j w[m][j] F_j - wd[m] fi_m;
 *   u_m = solve(alpha_m, beta_m);  fi_out_m = f_I(u_m).
 * node_coef is HOST memory [M][M + 4] = (w[m][0..M-1], wd[m], alpha_m,
 * alpha_m*phibar, alpha_m^2*phibar) with w = dt*q, wd = dt*d_m.  fe/fi are
 * [M][3C] with element stride fe_stride/fi_stride states (0 = every node
 * aliases the step-start slot, as after initialize_sweep, core.py:165-174);
 * first != 0 means fi_j = f_I(u0) computed inline (fi ignored).  u_out and
 * fi_out hold `count` states; neither may alias u0, fe or fi (nodes are
 * updated concurrently).  Replaces diagonal_sweep phase one plus the
 * solve/f_I half of _refresh_node (integrators.py:233-288); f_E of u_out is a
 * separate sdcsw_f_expl call.  Bit-identical to the reference arithmetic. */
int sdcsw_sweep_nodes(sdcsw_plan* plan, int n_nodes, int node_lo, int count,
                      const double* node_coef, const double* u0, const double* fe,
                      long long fe_stride, const double* fi, long long fi_stride, int first,
                      double* u_out, double* fi_out, void* stream);

/* sdcsw_sweep_nodes with the collocation-residual norm fused into the same
 * kernel (M <= 6, one state, unsplit plan): for every node m of the block,
 *   resid[q][f] = || u0 + sum_j w[m][j] (fe_j + fi_j) - u_prev[q] ||_2
 * per field f (Phi', zeta, delta) over the stored complex coefficients, where
 * u_prev holds the previous iterate's node values u_m (count states) - the
 * residual of the iterate whose tendencies fe/fi are.  resid is DEVICE memory
 * [count][3]; the reduction order is fixed (deterministic).  u_out / fi_out
 * are exactly those of sdcsw_sweep_nodes.  The reference monitors no residual
 * (its sweeps run a fixed count, integrators.py:347-381); this is the
 * north-star's fused quadrature + update + residual kernel.  The reduction
 * workspace is allocated with the plan and shared by its calls: residual sweeps
 * on one plan must be serialised on one stream.  Graph-capturable. */
int sdcsw_sweep_nodes_residual(sdcsw_plan* plan, int n_nodes, int node_lo, int count,
                               const double* node_coef, const double* u0, const double* fe,
                               long long fe_stride, const double* fi, long long fi_stride, int first,
                               const double* u_prev, double* u_out, double* fi_out, double* resid,
                               void* stream);

/* Closing last-node solve of a diagonal step (integrators.py:291-311):
 *   beta = u0 + sum_j (w[j] fe_j + w[j] fi_j) - wd fi_last ; u_out = solve.
 * final_coef is HOST memory [M + 4] = (w[0..M-1], wd, alpha, alpha*phibar,
 * alpha^2*phibar).  u_out may alias u0. */
/* One serial SDC sweep (all M nodes in order) on a single state: the
 * reference's serial_sweep (integrators.py:183-230, Alg. 1 / Eq. 5).  coef is
 * the serial stepper's coefficient block (W = dt q [M][M], dt explicit
 * weights [M], dt dtau [M], solve scalars [M][3]; serial_step_coefficients in
 * integrators.py of this package).  fe_old / fi_old: the previous iterate's
 * node tendencies (element stride fe_stride / fi_stride states; the first
 * sweep passes f_E(u0) with stride 0, and fi_old is ignored - f_I(u0) is
 * formed in the kernels).  Writes the new node tendencies fe_new / fi_new (M
 * states each) and node M's state u_last; work is caller-owned scratch of
 * M + 2 states.  The same kernels in the same order as the serial stepper
 * (bit-identical).  Uses the plan's API operand and workspaces: serialise
 * calls on one plan. */
int sdcsw_serial_sweep(sdcsw_plan* plan, int n_nodes, const double* coef, const double* u0,
                       const double* fe_old, long long fe_stride, const double* fi_old,
                       long long fi_stride, int first, double* fe_new, double* fi_new,
                       double* u_last, double* work, void* stream);

int sdcsw_final_node(sdcsw_plan* plan, int n_nodes, const double* final_coef, const double* u0,
                     const double* fe, long long fe_stride, const double* fi, long long fi_stride,
                     int first, double* u_out, void* stream);

/* Device-resident stepper owning all sweep storage and a CUDA graph of one
 * step.  mode 0 = diagonal SDC (dsdc_step, integrators.py:347-381),
 * mode 1 = serial SDC (sdc_step_serial, integrators.py:317-344).
 * coef is HOST memory:
 *   mode 0: [K-1][M][M+4] sweep node_coef blocks, then [M+4] final_coef;
 *   mode 1: [M][M] w = dt*q, then [M] explicit correction weights dt*ew,
 *           [M] implicit correction weights dt*dtau, [M][3] solve coefs. */
int sdcsw_stepper_create(sdcsw_plan* plan, int mode, int n_nodes, int n_sweeps,
                         const double* coef, int n_coef, sdcsw_stepper** out);
/* Ensemble variant: `members` independent states advanced together (BASELINE
 * config 4); u holds `members` consecutive states and every f_E carries
 * members x nodes GEMM columns.  Plan max_batch must be >= members x nodes.
 * Mode 0 only for members > 1. */
int sdcsw_stepper_create_ensemble(sdcsw_plan* plan, int mode, int n_nodes, int n_sweeps,
                                  int members, const double* coef, int n_coef,
                                  sdcsw_stepper** out);
int sdcsw_stepper_destroy(sdcsw_stepper* st);

/* Advance the device state u (one state, in place) by n_steps steps on
 * stream.  use_graph != 0 replays a captured CUDA graph per step.  The
 * per-step finiteness check of integrate (integrators.py:538-548,
 * core.py:42-50) runs on the device; read it with sdcsw_stepper_diverged. */
int sdcsw_stepper_run(sdcsw_stepper* st, double* u, int n_steps, int use_graph, void* stream);

/* First one-based step index (counted since the last reset) whose state was
 * non-finite, or 0.  Synchronises the stepper's stream. */
int sdcsw_stepper_diverged(sdcsw_stepper* st, int* step_index);
int sdcsw_stepper_reset(sdcsw_stepper* st, void* stream);

/* option 0: concurrent node chains per sweep (1..M); option 1: sequential
 * node updates (1 = the DIAGONAL_SEQUENTIAL analogue: one node at a time on
 * one stream); option 2: node updates fused into the analysis epilogue (1 =
 * on, the default for dSDC with one member, M <= 6 and the latency-regime
 * analysis; takes effect with chains = 1 and sequential = 0); option 3: steps
 * per replayed CUDA graph (1..64, default 8; programmatic dependent launch then
 * also overlaps step boundaries).  Bit-identical results in every setting.
 * Rebuilds the step graph. */
int sdcsw_stepper_set_option(sdcsw_stepper* st, int option, int value);

/* One step launched stage by stage with CUDA events (no graph) for the cost
 * model (perfmodel.fit_costs, pkg/src/parsdc/perfmodel.py:78-111): stage_ms =
 * [init, sweep 1 .. sweep K-1, final node] for dSDC, [init, sweep 1 .. K] for
 * serial SDC; n >= K + 1.  Synchronises. */
int sdcsw_stepper_profile(sdcsw_stepper* st, double* u, double* stage_ms, int n, void* stream);

/* One step stage by stage (as sdcsw_stepper_profile, one member) with a host
 * callback after every sweep: hook(user, k) runs after sweep k (dSDC: k = 1 ..
 * K-1, before the closing solve; serial SDC: k = 1 .. K) has completed on the
 * device, before the next sweep is enqueued, so the callback may read the
 * sweep's buffers (sdcsw_stepper_sweep_state).  stage_ms (optional, n >= K+1)
 * as sdcsw_stepper_profile.  Replaces the on_sweep(k, state) callback of
 * dsdc_step / sdc_step_serial (integrators.py:317-381).  Synchronises. */
typedef void (*sdcsw_sweep_hook)(void* user, int sweep);
int sdcsw_stepper_step_hooked(sdcsw_stepper* st, double* u, sdcsw_sweep_hook hook, void* user,
                              double* stage_ms, int n, void* stream);
/* Device buffers holding sweep k's tendencies (valid inside the hook of sweep
 * k): fe0 = f_E(u0) (one state), fe / fi = f_E, f_I of the M nodes (M
 * consecutive states).  The node states themselves are not retained (the
 * reference drops them too, integrators.py:233-246); f_I(u0) is recomputed. */
int sdcsw_stepper_sweep_state(sdcsw_stepper* st, int sweep, void** fe0, void** fe, void** fi);
/* Sweep storage of the stepper (the analogue of the reference's storage
 * accounting, tests/test_acceptance.py:284-305): bytes of device memory it owns
 * and the number of state-sized buffers among them (per member: fe0 and two
 * generations of the M nodes' fe, fi = 1 + 4M; plus node states where an f_E
 * reads them, and the serial-SDC quadrature / correction). */
int sdcsw_stepper_storage(sdcsw_stepper* st, long long* bytes, long long* state_buffers);

/* Number of kernels one step launches (for the bench's gpu_launches). */
int sdcsw_stepper_launches_per_step(sdcsw_stepper* st, int* n);

/* One stage of f_E on the plan's internal workspaces, for per-kernel timing
 * and stage-level parity tests: stage 0 = Legendre synthesis (u -> Fourier
 * workspace), 1 = ring FFT + products (Fourier -> analysis workspace),
 * 2 = Legendre analysis (analysis workspace -> out), 3 = synthesis from the
 * operand stage 0 prepared, 4 = analysis with the dSDC step's fused
 * node-update epilogue (nb nodes; in = u0, out = their f_I, updated in place;
 * zero coefficients - for timing the kernel the step runs).  `in`/`out` are
 * ignored where the stage reads/writes a workspace.  sdcsw_f_expl is stages
 * 0, 1, 2 back to back. */
int sdcsw_transform_stage(sdcsw_plan* plan, int stage, const double* in, double* out, int nb,
                          void* stream);

/* Device pointers and sizes of the internal workspaces: which 0 = Fourier
 * coefficients [max_batch][nlat/2][T+1][4 (U,V,zeta,Phi)][2 (N,S)] complex,
 * which 1 = analysis data, [max_batch][T+1] blocks of nlat/2 x 28 doubles:
 * [nlat/2][2 (N+S, N-S)][7 slots] complex when T < 400, in DMMA-fragment
 * order for the table-streaming analysis (T >= 400; gan_off in internal.cuh). */
int sdcsw_workspace(sdcsw_plan* plan, int which, void** ptr, long long* bytes);

/* Transform family of the plan: *kind = 0 when f_E contracts with the P and H
 * tables; 1 when it runs H-free (table-streaming plans, T >= 200 or ensembles,
 * unless SDCSW_PONLY=0 at plan creation): P to degree T+1 and the derivative
 * recurrence H_n = (n+1) eps_n P_{n-1} - n eps_{n+1} P_{n+1} on the coefficients,
 * 9 instead of 13 transforms per f_E.  The analysis workspace (which 1) then
 * holds 5 slots per (m, pair, fold): [m][nlat/2 / 4][2][4][5] complex.  Both
 * compute the reference's f_expl (problems/swe.py:174-205 restated on the sphere)
 * to rounding; *rows = packed table rows streamed per analysis/synthesis. */
int sdcsw_plan_transform_kind(sdcsw_plan* plan, int* kind, int* rows);

/* Spectral split (more GPUs than collocation nodes): the plan's
 * wavenumbers are partitioned over the S ranks of a spectral group, pairs
 * (m, T-m) dealt round-robin, and this rank keeps part sp.  Afterwards
 * sdcsw_sweep_nodes / sdcsw_final_node touch only own-m coefficients, and f_E
 * runs as begin (operand prep + synthesis of own m into part sp of `fourier`,
 * a caller-owned part-major buffer [S][nb][nlat/2][Lp][4][2] complex) ->
 * caller all-gathers the S parts of `fourier` (NCCL) -> end (ring kernel over
 * all latitudes + analysis of own m into fe).  S = 1 restores the unsplit plan.
 * The per-m and per-latitude arithmetic is unchanged, so results are
 * bit-identical to the unsplit plan.  Replaces nothing in the reference (its
 * space parallelism is scipy.fft worker threads, problems/swe.py:148-153). */
int sdcsw_plan_set_split(sdcsw_plan* plan, int S, int sp, void* fourier, long long bytes);
int sdcsw_split_info(sdcsw_plan* plan, int* Lp, int* n_own_m, int* n_own_idx);
int sdcsw_split_f_expl_begin(sdcsw_plan* plan, const double* u, int nb, void* stream);
int sdcsw_split_f_expl_end(sdcsw_plan* plan, double* fe, int nb, void* stream);

/* Node-parallel dSDC over peer memory (replaces the reference's
 * per-sweep thread-pool barrier, integrators.py:278-288, and the all-gather of
 * the node tendencies).  One exchange object per rank (one process per GPU):
 * rank r owns the contiguous node block [r P, min((r+1) P, M)), P = ceil(M /
 * world).  Per full sweep the rank solves its nodes, evaluates their f_E, and
 * the analysis kernel's epilogue stores (f_E, f_I) of its nodes straight into
 * every rank's exchange buffer over NVLink (option 0 = 0: a copy kernel after
 * a plain analysis instead); the next node kernel of every rank first posts
 * the exchange number into every rank's flag word (system-scope atomic, after
 * the publishing grid completed) and spins (acquire) until all ranks posted.
 * The closing last-node solve and the next f_E(u0) run redundantly on every
 * rank, so the state stays replicated and bit-identical to one GPU.  No NCCL
 * call on the data path.
 *   create: coef as sdcsw_stepper_create (mode 0); world <= 16.
 *   ipc_handle / open_peers: export this rank's buffer (a cudaIpcMemHandle_t,
 *     SDCSW_IPC_HANDLE_BYTES bytes) and open the handles of all ranks
 *     (world x SDCSW_IPC_HANDLE_BYTES, rank order; the own entry is skipped).
 *   base / attach_peer: the same for peers that live in this process
 *     (device pointers of other exchange objects, peer access enabled).
 *   create_split: world = G node groups x S spectral parts (rank = g S + sp,
 *     G <= M when S > 1).  The exchange splits the plan (sdcsw_plan_set_split
 *     with its own peer-mapped Fourier buffer); the state is m-partitioned
 *     (own wavenumbers valid).  Each f_E's split synthesis stores its part into
 *     every spectral peer's Fourier buffer and the ring kernel posts and waits
 *     for all parts before reading them; the node exchange runs among the G
 *     ranks sharing part sp.  create = create_split with S = 1.
 *   phase: enqueue one half-phase of a step on u - for f_E k = 0..K-1 (k = 0:
 *     f_E(u0), with the operand prep at phase 0; k >= 1: full sweep k,
 *     publishing node exchange k) phase 2k = [node kernel k] + synthesis and
 *     2k + 1 = ring + analysis; phase 2K = closing solve.  Phases 2k (k >= 2)
 *     and 2K wait for node exchange k - 1; phases 2k + 1 of a split exchange
 *     wait for the Fourier exchange of f_E k.
 *   post: enqueue only a post (idempotent): channel 0 = node exchange k of the
 *     current step, channel 1 = the next Fourier exchange.  A driver of
 *     several ranks on ONE stream posts for every rank before any rank's
 *     phase that waits, so no wait depends on a later kernel.
 *   run: n_steps steps (operand prep first); use_graph replays a captured
 *     graph of up to 8 steps.
 *   option 0: publish fused into the analysis epilogue (default 1 where the
 *     plan supports it: spherical, T < 400, unsplit).
 *   option 1: bound, in milliseconds, of every device wait on a peer's post
 *     (default 30000).  A wait that runs out records the peer and exchange
 *     and returns; later waits of the exchange do not wait again (the state
 *     is then invalid).  sdcsw_exchange_diverged reports it as
 *     SDCSW_ERR_PEER naming the rank - a dead or stalled peer produces an
 *     error, never a hung GPU.  reset clears it.
 *   info: own node block and kernels per step.
 *   reset: divergence is reported relative to the step count at the reset.
 * Every rank must run the same number of steps (the exchange numbers derive
 * from a device step counter that is never reset, so they stay in lock step);
 * a rank with no nodes still posts every exchange. */
#define SDCSW_IPC_HANDLE_BYTES 64
typedef struct sdcsw_exchange sdcsw_exchange;
int sdcsw_exchange_create(sdcsw_plan* plan, int n_nodes, int n_sweeps, const double* coef,
                          int n_coef, int world, int rank, sdcsw_exchange** out);
int sdcsw_exchange_create_split(sdcsw_plan* plan, int n_nodes, int n_sweeps, const double* coef,
                                int n_coef, int world, int rank, int spectral_parts,
                                sdcsw_exchange** out);
int sdcsw_exchange_ipc_handle(sdcsw_exchange* x, void* handle, int bytes);
int sdcsw_exchange_open_peers(sdcsw_exchange* x, const void* handles, int bytes_each);
int sdcsw_exchange_base(sdcsw_exchange* x, void** base);
int sdcsw_exchange_attach_peer(sdcsw_exchange* x, int peer, void* base);
int sdcsw_exchange_phase(sdcsw_exchange* x, double* u, int phase, void* stream);
int sdcsw_exchange_post(sdcsw_exchange* x, int channel, int k, void* stream);
int sdcsw_exchange_run(sdcsw_exchange* x, double* u, int n_steps, int use_graph, void* stream);
int sdcsw_exchange_set_option(sdcsw_exchange* x, int option, int value);
int sdcsw_exchange_info(sdcsw_exchange* x, int* node_lo, int* node_count, int* launches_per_step);
int sdcsw_exchange_diverged(sdcsw_exchange* x, int* step_index);
int sdcsw_exchange_reset(sdcsw_exchange* x, void* stream);
int sdcsw_exchange_destroy(sdcsw_exchange* x);

/* NCCL transport (SURVEY 8b "sdcsw_comm_init_all" / "sdcsw_allgather_rhs";
 * replaces the reference's per-sweep barrier over the node futures,
 * integrators.py:278-288, when the nodes of a sweep live on different GPUs).
 *   unique_id: rank 0 creates the NCCL unique id (SDCSW_COMM_ID_BYTES bytes);
 *     the caller carries it to every rank (torch.distributed bootstrap only).
 *   create: one communicator per process (ncclCommInitRank) on `device`.
 *   split: sub-communicator of the ranks passing the same color, ordered by
 *     key (ncclCommSplit) - node groups (same spectral part) and spectral
 *     groups (same node group) of the node x spectral partition.
 *   allgather_rhs: recv[world][count] <- every rank's send[count] doubles
 *     (ncclAllGather; in rank order), stream-ordered and graph-capturable.
 *     The node-parallel step gathers the (f_E, f_I) pairs of every rank's
 *     node block once per sweep, and the Fourier parts once per f_E of a
 *     spectral split.
 *   nccl_version: the loaded library's NCCL_VERSION_CODE. */
#define SDCSW_COMM_ID_BYTES 128
typedef struct sdcsw_comm sdcsw_comm;
int sdcsw_comm_unique_id(void* id, int bytes);
int sdcsw_comm_create(const void* id, int bytes, int world, int rank, int device, sdcsw_comm** out);
/* single-process multi-GPU (ncclCommInitAll): out[i] is rank i on devs[i] */
int sdcsw_comm_init_all(int ndev, const int* devs, sdcsw_comm** out);
int sdcsw_comm_split(sdcsw_comm* parent, int color, int key, sdcsw_comm** out);
int sdcsw_comm_info(sdcsw_comm* comm, int* world, int* rank);
int sdcsw_allgather_rhs(sdcsw_comm* comm, const double* send, double* recv, long long count,
                        void* stream);
int sdcsw_comm_destroy(sdcsw_comm* comm);
int sdcsw_nccl_version(void);

/* out = x + w * y over n doubles, rounded as numpy's `x + w * y` (product, then
 * sum); out may alias x.  The vector update of the reference schemes
 * imex_o2_step / ab2_si_step (integrators.py:387-420). */
int sdcsw_axpy(long long n, const double* x, double w, const double* y, double* out, void* stream);

/* Any non-finite entry among n doubles -> *flag = 1 (device int).
 * Replaces check_finite (core.py:42-50) without a host round trip. */
int sdcsw_check_finite(const double* x, long long n, int* flag, void* stream);

/* Bounds check of the library's own device allocations.  With SDCSW_GUARD=1 in
 * the environment when the library is loaded, every plan / stepper allocation
 * carries a 64 KiB canary in front and behind; this call synchronises the
 * device and returns the number of canary bytes any kernel has overwritten
 * (live allocations now, plus those found when allocations were freed) and the
 * number of live guarded allocations (-1: guards are off).  The reference has
 * no counterpart (numpy bounds-checks every index); it stands in for
 * compute-sanitizer memcheck in the tests (tests/test_gpu_guard.py). */
int sdcsw_guard_check(long long* corrupted_bytes, int* live_allocations);
/* Writes one byte past a 256-byte guarded allocation and frees it: with guards
 * on, the next sdcsw_guard_check reports one more corrupted byte (the proof
 * that the canaries see an overrun). */
int sdcsw_guard_selftest(void);

const char* sdcsw_last_error(void);
int sdcsw_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SDCSW_H */
