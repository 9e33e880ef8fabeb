"""Node-partitioned dSDC across processes (world size 2, gloo, CPU): the
orchestration of paper_2403_20135_b200.parallel_nodes with a numpy backend
reproduces the single-process oracle step bit-for-bit (the analogue of the
reference's thread-count invariance, pkg/tests/test_integrators.py:190-225)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class NumpyNodeBackend:
    """The node arithmetic of oracle/sdc.py behind the backend interface."""

    def __init__(self, prob):
        self.p = prob
        self.S = prob.state_size

    def empty(self, n):
        return torch.zeros((n, self.S), dtype=torch.complex128)

    def _state(self, t, j, stride):
        flat = t.reshape(-1)
        return flat[j * stride * self.S : j * stride * self.S + self.S].numpy()

    def f_expl(self, u, out, nb):
        uu = u.reshape(-1, self.S)
        for b in range(nb):
            out[b] = torch.from_numpy(self.p.f_expl(uu[b].numpy()))

    def sweep_nodes(self, m_count, lo, count, coef, u0, fe, fes, fi, fis, first, u_out, fi_out):
        u0n = u0.reshape(-1).numpy()
        fi0 = self.p.f_impl(u0n)
        fes_ = [self._state(fe, j, fes) for j in range(m_count)]
        fis_ = [fi0 if first else self._state(fi, j, fis) for j in range(m_count)]
        F = [fes_[j] + fis_[j] for j in range(m_count)]
        for q in range(count):
            m = lo + q
            c = coef[m * (m_count + 4) : (m + 1) * (m_count + 4)]
            acc = u0n.copy()
            for j in range(m_count):
                acc += c[j] * F[j]
            acc -= c[m_count] * fis_[m]
            u = self.p.implicit_solve(c[m_count + 1], acc)
            u_out[q] = torch.from_numpy(u)
            fi_out[q] = torch.from_numpy(self.p.f_impl(u))

    def final_node(self, m_count, coef, u0, fe, fes, fi, fis, first, u_out):
        u0n = u0.reshape(-1).numpy().copy()
        fi0 = self.p.f_impl(u0n)
        acc = u0n.copy()
        last = None
        for j in range(m_count):
            e = self._state(fe, j, fes)
            f = fi0 if first else self._state(fi, j, fis)
            acc += coef[j] * e
            acc += coef[j] * f
            last = f
        acc -= coef[m_count] * last
        u = self.p.implicit_solve(coef[m_count + 1], acc)
        u_out.reshape(-1)[:] = torch.from_numpy(u)


def _worker(rank, world, port, m_count, k_count, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.sphere_swe import SphericalShallowWaterOracle
    from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode
    from paper_2403_20135_b200.parallel_nodes import NodeParallelDsdc
    from paper_2403_20135_b200.sphere import SphereGrid, random_initial_state

    g = SphereGrid(trunc=10, nlat=16, nlon=32)
    prob = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    cfg = SdcConfig(table=CollocationTable.radau_right(m_count), n_sweeps=k_count,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=min(world, m_count))
    stepper = NodeParallelDsdc(NumpyNodeBackend(prob), cfg, 900.0, prob.phibar, prob.state_size)
    u = torch.from_numpy(random_initial_state(g, 5)).reshape(1, -1).clone()
    for _ in range(2):
        stepper.step(u)
    np.save(out_path + f".{rank}.npy", u.reshape(-1).numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m_count,k_count", [(2, 4, 3), (2, 3, 3), (2, 3, 1)])
def test_node_partition_matches_single_process(tmp_path, world, m_count, k_count):
    from oracle import sdc as osdc
    from oracle.sphere_swe import SphericalShallowWaterOracle
    from paper_2403_20135_b200 import CollocationTable
    from paper_2403_20135_b200.sphere import SphereGrid, random_initial_state

    port = 29500 + (os.getpid() % 1000)
    out = str(tmp_path / "u")
    mp.spawn(_worker, args=(world, port, m_count, k_count, out), nprocs=world, join=True)
    g = SphereGrid(trunc=10, nlat=16, nlon=32)
    prob = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    table = CollocationTable.radau_right(m_count)
    ref = random_initial_state(g, 5)
    for _ in range(2):
        ref = osdc.dsdc(prob, ref, 900.0, table, k_count)
    for r in range(world):
        got = np.load(out + f".{r}.npy")
        assert np.array_equal(got, ref), (r, np.abs(got - ref).max())
