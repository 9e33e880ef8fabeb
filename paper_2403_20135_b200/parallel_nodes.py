"""Node- and spectrally-parallel diagonal SDC across GPUs (one process per GPU).

The M node updates of a diagonal sweep are independent
(``pkg/src/parsdc/integrators.py:254-267``, paper Alg. 2); the reference runs
them on a thread pool with a per-sweep barrier (``:278-288``).  Here rank r of
a group of G processes owns the contiguous node block
``[r P, min((r+1) P, M))`` with ``P = ceil(M / G)``; per full sweep each rank

1. assembles beta and solves its own nodes (``sdcsw_sweep_nodes``),
2. evaluates f_E of its nodes (``sdcsw_f_expl``, nodes batched),
3. all-gathers the (fe, fi) pairs of every node - the one exchange step
   (``sdcsw_allgather_rhs``: NCCL over NVLink called from ``libsdcsw.so``,
   :mod:`.comm`; torch.distributed over gloo in the CPU tests),

after which every rank holds all tendencies, so the closing last-node solve
and the next step's f_E(u0) are computed redundantly and the state stays
replicated and bit-identical to the single-GPU run (the node arithmetic does
not depend on placement, exactly as the reference's thread-count invariance,
``pkg/tests/test_integrators.py:190-225``).

Gathered layout: ``G[world * P][2][S]`` (node-major; fe then fi), so node j's
fe is ``G + 2 j S`` and its fi ``G + (2 j + 1) S`` - the sweep kernels take
these with element stride 2 states.  The compute backend is pluggable:
:class:`CudaNodeBackend` calls ``libsdcsw.so``; tests supply a numpy backend.

With more GPUs than nodes the G ranks form NG node groups of
S spectral parts (G = NG S, rank r -> node group r // S, part r % S).  Part
sp owns the wavenumbers of pairs (m, T-m) dealt round-robin
(:func:`spectral_parts`); the state is m-partitioned, so node kernels,
synthesis and analysis touch own-m coefficients only, and each f_E adds one
all-gather of the synthesised Fourier coefficients inside the spectral group
(the ring FFTs need every m of a latitude).  The (fe, fi) all-gather runs in
the node-group communicator (same part, different node groups).  Every per-m
and per-latitude operation is unchanged, so results stay bit-identical.
"""

import math

import numpy as np

from .errors import ParameterError
from .integrators import diagonal_step_coefficients


def spectral_parts(trunc, n_parts):
    """part[m] for m = 0..T: pairs (m, T - m) dealt round-robin (as sdcsw_plan_set_split)."""
    part = [0] * (trunc + 1)
    i, m = 0, 0
    while m <= trunc - m:
        part[m] = part[trunc - m] = i % n_parts
        i += 1
        m += 1
    return part


def node_block(n_nodes, world, rank):
    """(lo, count, per_rank) of the contiguous node block owned by ``rank``."""
    per = math.ceil(n_nodes / world)
    lo = min(rank * per, n_nodes)
    count = max(0, min(per, n_nodes - lo))
    return lo, count, per


class CudaNodeBackend:
    """Device operations of one rank, through the C ABI."""

    def __init__(self, problem):
        self.problem = problem
        self.lib = problem._lib
        self.fourier = None

    def set_split(self, n_parts, part, max_batch):
        """Partition the plan's wavenumbers; returns the part-major Fourier buffer."""
        import ctypes

        import torch

        from . import _native

        p = self.problem
        if n_parts == 1:
            _native.check(self.lib.sdcsw_plan_set_split(p.handle, 1, 0, None, 0))
            self.fourier = None
            return None
        counts = [0] * n_parts
        for q in spectral_parts(p.trunc, n_parts):
            counts[q] += 1
        lp = max(counts)
        j = p.grid.nlat // 2
        self.fourier = torch.zeros((n_parts, max_batch * j * lp * 8), dtype=torch.complex128,
                                   device=p.device)
        _native.check(self.lib.sdcsw_plan_set_split(p.handle, n_parts, part, self.fourier.data_ptr(),
                                                    self.fourier.numel() * 16), "sdcsw_plan_set_split")
        self._part_elems = max_batch * j * lp * 8
        self._j, self._lp = j, lp
        return self.fourier

    def f_expl_split(self, u, out, nb, gather):
        """Split f_E: own-m synthesis, all-gather of the Fourier parts, ring + own-m analysis."""
        from . import _native

        p = self.problem
        _native.check(self.lib.sdcsw_split_f_expl_begin(p.handle, u.data_ptr(), nb, p.stream()))
        per = nb * self._j * self._lp * 8  # the kernels index parts with the call's batch
        flat = self.fourier.view(-1)
        parts = [flat[q * per : (q + 1) * per] for q in range(self.fourier.shape[0])]
        gather(parts)
        _native.check(self.lib.sdcsw_split_f_expl_end(p.handle, out.data_ptr(), nb, p.stream()))

    def empty(self, n_states):
        return self.problem.empty_states(n_states)

    def stream(self):
        return self.problem.stream()

    def make_comms(self, group, n_parts):
        """(node-group, spectral-group) NCCL communicators of the C ABI: one
        world communicator bootstrapped over ``group`` (unique id broadcast),
        split by spectral part (node groups) and by node group (spectral
        groups, only when ``n_parts`` > 1)."""
        from .comm import NcclComm

        world = NcclComm.bootstrap(self.problem.device.index, group)
        if n_parts == 1:
            return world, None
        part, ng = world.rank % n_parts, world.rank // n_parts
        node = world.split(part, ng)
        spec = world.split(ng, part)
        self._world_comm = world  # parent kept alive with its splits
        return node, spec

    def f_expl(self, u, out, nb):
        self.problem.f_expl_device(u, out, nb)

    def sweep_nodes(self, n_nodes, lo, count, coef, u0, fe, fe_stride, fi, fi_stride, first,
                    u_out, fi_out):
        from . import _native

        _native.check(
            self.lib.sdcsw_sweep_nodes(
                self.problem.handle, n_nodes, lo, count, _native.dptr(coef), u0.data_ptr(),
                fe.data_ptr(), fe_stride, fi.data_ptr(), fi_stride, int(first), u_out.data_ptr(),
                fi_out.data_ptr(), self.problem.stream(),
            ),
            "sdcsw_sweep_nodes",
        )

    def sweep_nodes_residual(self, n_nodes, lo, count, coef, u0, fe, fe_stride, fi, fi_stride,
                             first, u_prev, u_out, fi_out, resid):
        """sweep_nodes plus the fused per-(node, field) collocation-residual norms of the
        previous iterate (u_prev: its node values) into the device tensor resid [count, 3]."""
        from . import _native

        _native.check(
            self.lib.sdcsw_sweep_nodes_residual(
                self.problem.handle, n_nodes, lo, count, _native.dptr(coef), u0.data_ptr(),
                fe.data_ptr(), fe_stride, fi.data_ptr(), fi_stride, int(first), u_prev.data_ptr(),
                u_out.data_ptr(), fi_out.data_ptr(), resid.data_ptr(), self.problem.stream(),
            ),
            "sdcsw_sweep_nodes_residual",
        )

    def serial_sweep(self, n_nodes, coef, u0, fe_old, fe_stride, fi_old, fi_stride, first,
                     fe_new, fi_new, u_last, work):
        """One serial SDC sweep (``sdcsw_serial_sweep``; the reference's
        ``serial_sweep``, ``integrators.py:183-230``); ``work``: M + 2 states."""
        from . import _native

        _native.check(
            self.lib.sdcsw_serial_sweep(
                self.problem.handle, n_nodes, _native.dptr(coef), u0.data_ptr(), fe_old.data_ptr(),
                fe_stride, fi_old.data_ptr(), fi_stride, int(first), fe_new.data_ptr(),
                fi_new.data_ptr(), u_last.data_ptr(), work.data_ptr(), self.problem.stream(),
            ),
            "sdcsw_serial_sweep",
        )

    def final_node(self, n_nodes, coef, u0, fe, fe_stride, fi, fi_stride, first, u_out):
        from . import _native

        _native.check(
            self.lib.sdcsw_final_node(
                self.problem.handle, n_nodes, _native.dptr(coef), u0.data_ptr(), fe.data_ptr(),
                fe_stride, fi.data_ptr(), fi_stride, int(first), u_out.data_ptr(),
                self.problem.stream(),
            ),
            "sdcsw_final_node",
        )


class NodeParallelDsdc:
    """One dSDC step with nodes (and, with ``spectral_parts`` > 1, wavenumbers)
    partitioned over the ranks of ``group``."""

    def __init__(self, backend, cfg, dt, phibar, state_size, group=None, spectral_parts=1):
        import torch.distributed as dist

        self.backend = backend
        if dist.is_available() and dist.is_initialized():
            world, rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            world, rank = 1, 0
        S = int(spectral_parts)
        if S < 1 or world % S:
            raise ParameterError(f"{world} ranks do not split into spectral groups of {S}")
        self.nparts = S
        self.part = rank % S
        node_group_index = rank // S
        n_groups = world // S
        if hasattr(backend, "make_comms"):  # the device path: NCCL through the C ABI
            self.node_comm, self.spec_comm = backend.make_comms(group, S)
        else:  # CPU tests: torch.distributed collectives (gloo)
            from .comm import DistComm

            if S == 1:
                self.node_comm, self.spec_comm = DistComm(group), None
            else:
                # every rank must create every group, in the same order
                ranks = list(range(world)) if group is None else dist.get_process_group_ranks(group)
                node_groups = [dist.new_group([ranks[g * S + q] for g in range(n_groups)]) for q in range(S)]
                spec_groups = [dist.new_group([ranks[g * S + q] for q in range(S)]) for g in range(n_groups)]
                self.node_comm = DistComm(node_groups[self.part])
                self.spec_comm = DistComm(spec_groups[node_group_index])
        self._stream = getattr(backend, "stream", lambda: None)
        self.world = n_groups
        self.rank = node_group_index
        self.m = cfg.table.n_nodes
        self.k = cfg.n_sweeps
        self.lo, self.count, self.per = node_block(self.m, self.world, self.rank)
        self.S = state_size
        coef = diagonal_step_coefficients(cfg, dt, phibar)
        block = self.m * (self.m + 4)
        self.sweep_coef = [np.ascontiguousarray(coef[i * block : (i + 1) * block]) for i in range(self.k - 1)]
        self.final_coef = np.ascontiguousarray(coef[(self.k - 1) * block :])
        p = self.per
        self.fe0 = backend.empty(1)
        self.gathered = backend.empty(2 * self.world * p)  # [world*P][2][S]
        self.local = backend.empty(2 * p)                    # [P][2][S] own block
        self.ustage = backend.empty(max(1, p))
        self.fi_tmp = backend.empty(max(1, p))
        self.fe_tmp = backend.empty(max(1, p))
        if self.m > 16:
            raise ParameterError("at most 16 nodes")
        if self.nparts > 1:
            backend.set_split(self.nparts, self.part, max(p, 1))

    def _f_expl(self, u, out, nb):
        if self.nparts == 1:
            self.backend.f_expl(u, out, nb)
            return

        def gather(parts):  # the one Fourier exchange of a split f_E (one all-gather, in place)
            flat = self.backend.fourier.view(-1)[: len(parts) * parts[0].numel()]
            self.spec_comm.allgather(flat, parts[self.part], self._stream())

        self.backend.f_expl_split(u, out, nb, gather)

    def counts_per_step(self):
        """Per-rank work: own nodes only (the redundant init/final are counted once per rank)."""
        n = 1 + (self.k - 1) * self.count
        return n, n, (self.k - 1) * self.count + 1

    def close(self):
        for c in (self.node_comm, self.spec_comm, getattr(self.backend, "_world_comm", None)):
            if c is not None:
                c.close()

    def capture(self, u, n_steps=1):
        """A CUDA graph of ``n_steps`` steps on ``u`` (kernels and NCCL all-gathers
        replayed without host work); ``graph.replay()`` advances ``u`` in place."""
        import torch

        scratch = u.clone()
        self.step(scratch)  # lazy initialisation (NCCL communicators) outside the capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(n_steps):
                self.step(u)
        torch.cuda.synchronize()
        return graph

    def step(self, u):
        """Advance the replicated state tensor ``u`` (shape [1, S] or [S]) in place."""
        b = self.backend
        g = self.gathered
        self._f_expl(u, self.fe0, 1)
        fe_src, fe_stride = self.fe0, 0
        fi_src, fi_stride = self.fe0, 0
        first = True
        fe_view = g.view(-1)  # fe of node j at state offset 2j
        fi_view = g.view(-1)[self.S :]  # fi of node j at state offset 2j + 1
        for k in range(1, self.k):
            if self.count:
                b.sweep_nodes(self.m, self.lo, self.count, self.sweep_coef[k - 1], u, fe_src,
                              fe_stride, fi_src, fi_stride, first, self.ustage, self.fi_tmp)
                self._f_expl(self.ustage, self.fe_tmp, self.count)
                loc = self.local.view(self.per, 2, -1)
                loc[: self.count, 0].copy_(self.fe_tmp.view(-1, self.S)[: self.count])
                loc[: self.count, 1].copy_(self.fi_tmp.view(-1, self.S)[: self.count])
            self.node_comm.allgather(self.gathered.view(-1), self.local.view(-1), self._stream())
            fe_src, fe_stride = fe_view, 2
            fi_src, fi_stride = fi_view, 2
            first = False
        b.final_node(self.m, self.final_coef, u, fe_src, fe_stride, fi_src, fi_stride, first, u)
        return u


class PeerNodeParallelDsdc:
    """Node-parallel dSDC with the per-sweep exchange done by the kernels over
    peer memory (``sdcsw_exchange_*``, ``csrc/peer.cu``): the analysis epilogue
    of each rank stores (f_E, f_I) of its own nodes into every rank's exchange
    buffer through NVLink; the next node kernel posts the exchange number into
    every rank's flag word and waits until all ranks posted it - no NCCL call
    and no host synchronisation on the data path.  Same node
    partition and bit-identical results as :class:`NodeParallelDsdc`.

    ``group`` (torch.distributed) is used once, to exchange the CUDA IPC
    handles of the buffers; with ``world == 1`` no process group is needed."""

    def __init__(self, problem, cfg, dt, group=None, world=None, rank=None, fused=None,
                 exchange_handles=True, spectral_parts=1):
        import ctypes

        from . import _native

        self.problem = problem
        self.lib = problem._lib
        if world is None:
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized():
                world, rank = dist.get_world_size(group), dist.get_rank(group)
            else:
                world, rank = 1, 0
        self.world, self.rank = int(world), int(rank)
        self.nparts = int(spectral_parts)
        self.part = self.rank % self.nparts
        self.m = cfg.table.n_nodes
        self.k = cfg.n_sweeps
        scalars = getattr(problem, "solve_coefficients", None)
        self._coef = np.ascontiguousarray(
            diagonal_step_coefficients(cfg, dt, problem.mean_geopotential, scalars))
        handle = ctypes.c_void_p()
        _native.check(
            self.lib.sdcsw_exchange_create_split(problem.handle, self.m, self.k,
                                                 _native.dptr(self._coef), self._coef.size,
                                                 self.world, self.rank, self.nparts,
                                                 ctypes.byref(handle)),
            "sdcsw_exchange_create",
        )
        self.handle = handle
        if fused is not None:
            self.set_fused(fused)
        if self.world > 1 and exchange_handles:
            self.open_peers(group)

    def ipc_handle(self):
        """This rank's exchange-buffer IPC handle (bytes), or None if it cannot be exported."""
        import ctypes

        from . import _native

        mine = ctypes.create_string_buffer(_native.IPC_HANDLE_BYTES)
        st = self.lib.sdcsw_exchange_ipc_handle(self.handle, mine, _native.IPC_HANDLE_BYTES)
        return mine.raw if st == _native.SDCSW_OK else None

    def open_peers(self, group=None, mine=b""):
        """All-gather the IPC handles over ``group`` and map every peer's buffer.

        Collective: every rank of the group must call it, including a rank
        whose exchange could not be created (it passes ``mine=None`` through
        :meth:`join_failed`), so that a failure on some ranks never leaves the
        others blocked in the all-gather; returns False on every rank if any
        rank failed."""
        import ctypes

        import torch.distributed as dist

        from . import _native

        if mine == b"":
            mine = self.ipc_handle()
        every = [None] * self.world
        dist.all_gather_object(every, mine, group=group)
        if any(h is None for h in every):
            return False
        blob = ctypes.create_string_buffer(b"".join(every), self.world * _native.IPC_HANDLE_BYTES)
        _native.check(self.lib.sdcsw_exchange_open_peers(self.handle, blob, _native.IPC_HANDLE_BYTES),
                      "sdcsw_exchange_open_peers")
        return True

    @classmethod
    def create_collective(cls, problem, cfg, dt, spectral_parts=1, group=None):
        """Create the exchange on every rank of ``group`` and map the peers, or
        fail on ALL ranks together: returns ``(exchange, None)`` everywhere or
        ``(None, reason)`` everywhere (reason is this rank's own error, or that
        another rank failed).  Safe when creation or mapping fails on some ranks
        only: the one collective (the handle all-gather) is joined by every
        rank, and the outcome is agreed with a MIN all-reduce."""
        import torch
        import torch.distributed as dist

        x, err = None, None
        try:  # local part only (no collective inside)
            x = cls(problem, cfg, dt, group=group, spectral_parts=spectral_parts, exchange_handles=False)
        except Exception as exc:  # noqa: BLE001 - reported to the caller
            err = f"{type(exc).__name__}: {exc}"
        try:
            opened = x.open_peers(group, mine=x.ipc_handle()) if x is not None else cls.join_failed(group)
        except Exception as exc:  # noqa: BLE001 - a local mapping failure
            opened, err = False, f"{type(exc).__name__}: {exc}"
        dev = getattr(problem, "device", None)
        backend = dist.get_backend(group)
        ok = torch.tensor([1 if opened else 0], dtype=torch.int32,
                          device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()):
            return x, None
        if x is not None:
            x.close()
        return None, err or "peer exchange unavailable on another rank"

    @staticmethod
    def join_failed(group=None):
        """The collective part of :meth:`open_peers` for a rank whose exchange
        could not be created: contributes no handle, so every rank sees the
        failure and nobody opens peers."""
        import torch.distributed as dist

        every = [None] * dist.get_world_size(group)
        dist.all_gather_object(every, None, group=group)
        return False

    @classmethod
    def in_process(cls, problem, cfg, dt, world, fused=None, spectral_parts=1):
        """``world`` exchange objects of one process on one device, attached to
        each other directly (no IPC) - for driving several ranks' phases in
        stream order (:meth:`run_in_stream_order`).  ``problem`` is one problem
        or, with spectral parts (each rank splits its plan), one per rank."""
        import ctypes

        from . import _native

        probs = problem if isinstance(problem, (list, tuple)) else [problem] * world
        if spectral_parts > 1 and len({id(q) for q in probs}) != world:
            raise ParameterError("spectral parts need one problem (plan) per rank")
        ranks = [cls(probs[r], cfg, dt, world=world, rank=r, fused=fused, exchange_handles=False,
                     spectral_parts=spectral_parts)
                 for r in range(world)]
        bases = []
        for x in ranks:
            b = ctypes.c_void_p()
            _native.check(x.lib.sdcsw_exchange_base(x.handle, ctypes.byref(b)))
            bases.append(b)
        for x in ranks:
            for q, b in enumerate(bases):
                if q != x.rank:
                    _native.check(x.lib.sdcsw_exchange_attach_peer(x.handle, q, b),
                                  "sdcsw_exchange_attach_peer")
        return ranks

    def set_wait_bound(self, ms):
        """Bound (milliseconds) of every device wait on a peer's post; a wait that
        runs out makes :meth:`diverged` raise ``DeviceError`` naming the rank."""
        from . import _native

        _native.check(self.lib.sdcsw_exchange_set_option(self.handle, 1, int(ms)),
                      "sdcsw_exchange_set_option")

    def set_fused(self, on=True):
        """Publish from the analysis epilogue (default where supported) or by a copy kernel."""
        from . import _native

        _native.check(self.lib.sdcsw_exchange_set_option(self.handle, 0, int(bool(on))),
                      "sdcsw_exchange_set_option")

    def info(self):
        """(node_lo, node_count, kernels per step) of this rank."""
        import ctypes

        lo, cnt, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        self.lib.sdcsw_exchange_info(self.handle, ctypes.byref(lo), ctypes.byref(cnt), ctypes.byref(n))
        return lo.value, cnt.value, n.value

    def counts_per_step(self):
        """Per-rank evaluations (own nodes; the redundant init/final counted once per rank)."""
        _, count, _ = self.info()
        n = 1 + (self.k - 1) * count
        return n, n, (self.k - 1) * count + 1

    def phase(self, u, phase):
        """Enqueue one half-phase of a step on ``u`` (``sdcsw_exchange_phase``):
        2k = [node kernel k] + synthesis and 2k + 1 = ring + analysis of f_E k
        (k = 0: f_E(u0)), 2K = closing solve."""
        from . import _native

        _native.check(self.lib.sdcsw_exchange_phase(self.handle, u.data_ptr(), int(phase),
                                                    self.problem.stream()), "sdcsw_exchange_phase")

    def post(self, channel, k=0):
        """Enqueue only a post: channel 0 = node exchange ``k`` of the current
        step, channel 1 = the next Fourier exchange (spectral parts)."""
        from . import _native

        _native.check(self.lib.sdcsw_exchange_post(self.handle, int(channel), int(k),
                                                   self.problem.stream()), "sdcsw_exchange_post")

    @staticmethod
    def run_in_stream_order(ranks, states, n_steps):
        """Advance the in-process ranks (:meth:`in_process`) on one stream:
        before each half-phase every rank posts what the half-phase waits for,
        then every rank runs it - each wait is satisfied by earlier kernels."""
        k_sweeps = ranks[0].k
        split = ranks[0].nparts > 1
        # without spectral parts the ranks may share one plan (one workspace):
        # each rank then runs both halves of an f_E back to back
        groups = ([[h] for h in range(2 * k_sweeps + 1)] if split else
                  [[2 * k, 2 * k + 1] for k in range(k_sweeps)] + [[2 * k_sweeps]])
        for _ in range(n_steps):
            for hs in groups:
                k = hs[0] // 2
                if hs[0] % 2 == 0 and k >= 2:  # node kernel k / closing solve: node exchange k - 1
                    for x in ranks:
                        x.post(0, k - 1)
                if hs[0] % 2 == 1:  # (split) ring of f_E k: its Fourier exchange
                    for x in ranks:
                        if k == 0 or x.info()[1] > 0:
                            x.post(1)
                for x, u in zip(ranks, states):
                    for h in hs:
                        x.phase(u, h)

    def run_serialized(self, u, n_steps, group=None):
        """Advance ``u`` with the ranks of ``group`` (one process each) taking turns:
        before every half-phase each rank posts what that half-phase waits for
        (post-only kernels), then the ranks run the half-phase one after another
        with a host barrier in between - every wait is satisfied by completed
        kernels of the other processes, and no kernel ever waits on a running one
        (the B200 profiling guide forbids spinning kernels of several processes on
        one GPU).  Same data path as :meth:`run` otherwise: real CUDA-IPC
        mappings, stores into peer buffers, system-scope posts.  For testing the
        multi-process protocol on one GPU."""
        import torch
        import torch.distributed as dist

        k_sweeps = self.k
        split = self.nparts > 1
        groups = ([[h] for h in range(2 * k_sweeps + 1)] if split else
                  [[2 * k, 2 * k + 1] for k in range(k_sweeps)] + [[2 * k_sweeps]])
        world = dist.get_world_size(group)
        me = dist.get_rank(group)
        for _ in range(n_steps):
            for hs in groups:
                k = hs[0] // 2
                if hs[0] % 2 == 0 and k >= 2:
                    self.post(0, k - 1)
                if hs[0] % 2 == 1 and (k == 0 or self.info()[1] > 0):
                    self.post(1)
                torch.cuda.synchronize()
                dist.barrier(group)
                for turn in range(world):
                    if turn == me:
                        for h in hs:
                            self.phase(u, h)
                        torch.cuda.synchronize()
                    dist.barrier(group)

    def own_coefficients(self):
        """Boolean mask over one field's coefficients (m-major triangle): the
        entries this rank's state holds (all unless spectral parts)."""
        trunc = self.problem.trunc
        part = np.array(spectral_parts(trunc, self.nparts))
        ms = np.concatenate([np.full(trunc + 1 - m, m) for m in range(trunc + 1)])
        return part[ms] == self.part

    def run(self, u, n_steps, use_graph=True):
        """Advance the replicated device state ``u`` by ``n_steps`` steps in place."""
        from . import _native

        _native.check(self.lib.sdcsw_exchange_run(self.handle, u.data_ptr(), int(n_steps),
                                                  int(bool(use_graph)), self.problem.stream()),
                      "sdcsw_exchange_run")

    def reset(self):
        """Clear the divergence flag; later step indices count from here."""
        from . import _native

        _native.check(self.lib.sdcsw_exchange_reset(self.handle, self.problem.stream()),
                      "sdcsw_exchange_reset")

    def diverged(self):
        """First non-finite step index since creation / reset (0 = none); synchronises.
        Raises ``DeviceError`` if a peer did not post an exchange within the
        wait bound (:meth:`set_wait_bound`)."""
        import ctypes

        v = ctypes.c_int()
        from . import _native

        _native.check(self.lib.sdcsw_exchange_diverged(self.handle, ctypes.byref(v)))
        return v.value

    def close(self):
        if self.handle is not None:
            self.lib.sdcsw_exchange_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
