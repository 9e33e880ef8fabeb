"""Node-parallel diagonal SDC across GPUs (one process per GPU).

The M node updates of a diagonal sweep are independent
(``pkg/src/parsdc/integrators.py:254-267``, paper Alg. 2); the reference runs
them on a thread pool with a per-sweep barrier (``:278-288``).  Here rank r of
a group of G processes owns the contiguous node block
``[r P, min((r+1) P, M))`` with ``P = ceil(M / G)``; per full sweep each rank

1. assembles beta and solves its own nodes (``sdcsw_sweep_nodes``),
2. evaluates f_E of its nodes (``sdcsw_f_expl``, nodes batched),
3. all-gathers the (fe, fi) pairs of every node - the one exchange step
   (NCCL over NVLink on the GPU; gloo in the CPU tests),

after which every rank holds all tendencies, so the closing last-node solve
and the next step's f_E(u0) are computed redundantly and the state stays
replicated and bit-identical to the single-GPU run (the node arithmetic does
not depend on placement, exactly as the reference's thread-count invariance,
``pkg/tests/test_integrators.py:190-225``).

Gathered layout: ``G[world * P][2][S]`` (node-major; fe then fi), so node j's
fe is ``G + 2 j S`` and its fi ``G + (2 j + 1) S`` - the sweep kernels take
these with element stride 2 states.  The compute backend is pluggable:
:class:`CudaNodeBackend` calls ``libsdcsw.so``; tests supply a numpy backend.
"""

import math

import numpy as np

from .errors import ParameterError
from .integrators import diagonal_step_coefficients


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

    def empty(self, n_states):
        return self.problem.empty_states(n_states)

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
    """One dSDC step with nodes partitioned over the ranks of ``group``."""

    def __init__(self, backend, cfg, dt, phibar, state_size, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.backend = backend
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
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
        # views for all_gather: one chunk per rank
        self.chunks = list(self.gathered.view(self.world, 2 * p, -1).unbind(0))
        if self.m > 16:
            raise ParameterError("at most 16 nodes")

    def counts_per_step(self):
        """Per-rank work: own nodes only (the redundant init/final are counted once per rank)."""
        n = 1 + (self.k - 1) * self.count
        return n, n, (self.k - 1) * self.count + 1

    def step(self, u):
        """Advance the replicated state tensor ``u`` (shape [1, S] or [S]) in place."""
        b = self.backend
        g = self.gathered
        b.f_expl(u, self.fe0, 1)
        fe_src, fe_stride = self.fe0, 0
        fi_src, fi_stride = self.fe0, 0
        first = True
        fe_view = g.view(-1)  # fe of node j at state offset 2j
        fi_view = g.view(-1)[self.S :]  # fi of node j at state offset 2j + 1
        for k in range(1, self.k):
            if self.count:
                b.sweep_nodes(self.m, self.lo, self.count, self.sweep_coef[k - 1], u, fe_src,
                              fe_stride, fi_src, fi_stride, first, self.ustage, self.fi_tmp)
                b.f_expl(self.ustage, self.fe_tmp, self.count)
                loc = self.local.view(self.per, 2, -1)
                loc[: self.count, 0].copy_(self.fe_tmp.view(-1, self.S)[: self.count])
                loc[: self.count, 1].copy_(self.fi_tmp.view(-1, self.S)[: self.count])
            self.dist.all_gather(self.chunks, self.local, group=self.group)
            fe_src, fe_stride = fe_view, 2
            fi_src, fi_stride = fi_view, 2
            first = False
        b.final_node(self.m, self.final_coef, u, fe_src, fe_stride, fi_src, fi_stride, first, u)
        return u
