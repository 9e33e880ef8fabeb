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
    """The node arithmetic of oracle/sdc.py behind the backend interface; in
    split mode the oracle's f_E restated per owned wavenumber (same per-m
    numpy operations, so the gathered result is bit-identical)."""

    def __init__(self, prob):
        self.p = prob
        self.S = prob.state_size
        self.part_of = None

    def set_split(self, n_parts, part, max_batch):
        from paper_2403_20135_b200.parallel_nodes import spectral_parts

        p = self.p
        self.part_of = np.array(spectral_parts(p.trunc, n_parts))
        self.part = part
        self.own_m = np.nonzero(self.part_of == part)[0]
        self.nf = p.nlon // 2 + 1
        self.fourier = torch.zeros((n_parts, max_batch * p.nlat * self.nf * 4), dtype=torch.complex128)
        return self.fourier

    def _synth_own(self, coef, tab):
        p = self.p
        out = np.zeros((p.nlat, self.nf), dtype=complex)
        for m in self.own_m:
            sl = slice(p.bounds[m], p.bounds[m + 1])
            out[:, m] = coef[sl] @ tab[sl]
        return out

    def _anal_own(self, fourier, tab, weight, out):
        p = self.p
        wf = (2.0 * np.pi * weight)[:, None] * fourier
        for m in self.own_m:
            sl = slice(p.bounds[m], p.bounds[m + 1])
            out[sl] = tab[sl] @ wf[:, m]

    def f_expl_split(self, u, out, nb, gather):
        p = self.p
        c = p.n_coef
        per = p.nlat * self.nf * 4
        flat = self.fourier.view(-1)
        parts = [flat[q * nb * per : (q + 1) * nb * per] for q in range(self.fourier.shape[0])]
        uu = u.reshape(-1, self.S)
        mine = parts[self.part].view(nb, 4, p.nlat, self.nf)
        for b in range(nb):
            phi, zeta, delta = p.views(uu[b].numpy())
            a = p.radius
            psi, chi = -zeta * p.inv_lam, -delta * p.inv_lam
            im = 1j * p.m_of
            uf = (self._synth_own(im * chi, p.p) - self._synth_own(psi, p.h)) / a
            vf = (self._synth_own(im * psi, p.p) + self._synth_own(chi, p.h)) / a
            for f, arr in enumerate((uf, vf, self._synth_own(zeta, p.p), self._synth_own(phi, p.p))):
                mine[b, f] = torch.from_numpy(arr)
        gather(parts)
        for b in range(nb):
            full = np.zeros((4, p.nlat, self.nf), dtype=complex)
            for m in range(p.trunc + 1):
                q = self.part_of[m]
                full[:, :, m] = parts[q].view(nb, 4, p.nlat, self.nf)[b, :, :, m].numpy()
            uf, vf, zf, pf = full
            ug, vg = p.to_grid(uf), p.to_grid(vf)
            zg, pg = p.to_grid(zf), p.to_grid(pf)
            eta = zg + (2.0 * p.omega * p.mu)[:, None]
            fa, fb = p.to_fourier(eta * ug), p.to_fourier(eta * vg)
            fc, fd = p.to_fourier(pg * ug), p.to_fourier(pg * vg)
            fke = p.to_fourier((ug * ug + vg * vg) / (2.0 * p.coslat2)[:, None])
            wt = p.w / p.coslat2
            res = out.reshape(-1, self.S)[b].numpy()
            t = {k: np.zeros(c, dtype=complex) for k in ("cp", "dh", "ap", "bh", "bp", "ah", "ke")}
            self._anal_own(fc, p.p, wt, t["cp"])
            self._anal_own(fd, p.h, wt, t["dh"])
            self._anal_own(fa, p.p, wt, t["ap"])
            self._anal_own(fb, p.h, wt, t["bh"])
            self._anal_own(fb, p.p, wt, t["bp"])
            self._anal_own(fa, p.h, wt, t["ah"])
            self._anal_own(fke, p.p, p.w, t["ke"])
            im = 1j * p.m_of
            own = np.isin(p.m_of, self.own_m)
            div_mass = (im * t["cp"] - t["dh"]) / p.radius
            div_abs = (im * t["ap"] - t["bh"]) / p.radius
            curl_abs = (im * t["bp"] + t["ah"]) / p.radius
            vals = [-div_mass, -div_abs, curl_abs + p.lam * t["ke"]]
            for k in range(3):
                seg = vals[k]
                seg[p.m_of == 0] = seg[p.m_of == 0].real
                res[k * c : (k + 1) * c][own] = seg[own]

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


def _worker(rank, world, port, m_count, k_count, out_path, nparts=1):
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
    stepper = NodeParallelDsdc(NumpyNodeBackend(prob), cfg, 900.0, prob.phibar, prob.state_size,
                               spectral_parts=nparts)
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


def test_node_and_spectral_split_matches_single_process(tmp_path):
    """4 ranks = 2 node groups x 2 spectral parts: every rank owns
    half the wavenumbers; the assembled state equals the single-process oracle
    bit for bit."""
    from oracle import sdc as osdc
    from oracle.sphere_swe import SphericalShallowWaterOracle
    from paper_2403_20135_b200 import CollocationTable
    from paper_2403_20135_b200.parallel_nodes import spectral_parts
    from paper_2403_20135_b200.sphere import SphereGrid, random_initial_state

    world, nparts, m_count, k_count = 4, 2, 3, 3
    port = 29700 + (os.getpid() % 1000)
    out = str(tmp_path / "u")
    mp.spawn(_worker, args=(world, port, m_count, k_count, out, nparts), nprocs=world, join=True)
    g = SphereGrid(trunc=10, nlat=16, nlon=32)
    prob = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    table = CollocationTable.radau_right(m_count)
    ref = random_initial_state(g, 5)
    for _ in range(2):
        ref = osdc.dsdc(prob, ref, 900.0, table, k_count)
    part_of = np.array(spectral_parts(g.trunc, nparts))
    c = prob.n_coef
    for ng in range(world // nparts):
        got = np.zeros_like(ref)
        for q in range(nparts):
            st = np.load(out + f".{ng * nparts + q}.npy")
            own = np.tile(part_of[prob.m_of] == q, 3)
            got[own] = st[own]
        assert np.array_equal(got, ref), np.abs(got - ref).max()
    assert sorted(set(part_of.tolist())) == [0, 1]
    assert abs((part_of[prob.m_of] == 0).sum() - c / 2) <= g.trunc + 1


class _FakeExchangeLib:
    """Records the exchange calls of PeerNodeParallelDsdc (host logic only)."""

    def __init__(self, rank, fail_create=False):
        self.rank = rank
        self.calls = []
        self.fail_create = fail_create

    def sdcsw_exchange_create_split(self, plan, m, k, coef, n_coef, world, rank, parts, out):
        self.calls.append(("create", m, k, n_coef, world, rank, parts))
        if self.fail_create:
            return 2  # SDCSW_ERR_CUDA (e.g. the IPC buffer allocation failed)
        out._obj.value = 1000 + rank
        return 0

    def sdcsw_exchange_ipc_handle(self, h, buf, nbytes):
        import ctypes

        ctypes.memmove(buf, bytes([self.rank + 1]) * nbytes, nbytes)
        return 0

    def sdcsw_exchange_open_peers(self, h, blob, each):
        self.calls.append(("open", blob.raw, each))
        return 0

    def sdcsw_exchange_destroy(self, h):
        return 0


class _FakeProblem:
    handle = None
    mean_geopotential = 9.80616e4

    def __init__(self, rank, fail_create=False):
        self._lib = _FakeExchangeLib(rank, fail_create)


def _peer_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode
    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

    cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=3,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=1)
    prob = _FakeProblem(rank)
    x = PeerNodeParallelDsdc(prob, cfg, 90.0)
    create = prob._lib.calls[0]
    opened = prob._lib.calls[1]
    np.save(out_path + f".{rank}.npy", np.frombuffer(opened[1], dtype=np.uint8))
    assert create == ("create", 4, 3, x._coef.size, world, rank, 1), create
    assert x._coef.size >= 2 * 4 * 8 + 8
    assert x.handle.value == 1000 + rank
    dist.barrier()
    dist.destroy_process_group()


def test_peer_exchange_handles_gathered_in_rank_order(tmp_path):
    """PeerNodeParallelDsdc (world 3, gloo): every rank creates its exchange
    with (world, rank) and opens the IPC handles of all ranks in rank order."""
    world = 3
    port = 29900 + (os.getpid() % 97)
    out = str(tmp_path / "h")
    mp.spawn(_peer_worker, args=(world, port, out), nprocs=world, join=True)
    want = np.concatenate([np.full(64, q + 1, dtype=np.uint8) for q in range(world)])
    for r in range(world):
        assert np.array_equal(np.load(out + f".{r}.npy"), want)


def _peer_fail_worker(rank, world, port, bad, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode
    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

    cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=3,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=1)
    prob = _FakeProblem(rank, fail_create=rank in bad)
    x, err = PeerNodeParallelDsdc.create_collective(prob, cfg, 90.0)
    opened = any(c[0] == "open" for c in prob._lib.calls)
    with open(out_path + f".{rank}", "w") as f:
        f.write(f"{x is None} {opened} {err}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("bad", [(1,), (0, 2), ()])
def test_peer_exchange_failure_is_collective(tmp_path, bad):
    """if the exchange cannot be created on some ranks, every rank
    still joins the one collective and all of them fall back together (no
    hang, nobody opens peers); with no failure every rank opens its peers."""
    world = 3
    port = 29300 + (os.getpid() % 97) + 7 * len(bad)
    out = str(tmp_path / "f")
    mp.spawn(_peer_fail_worker, args=(world, port, bad, out), nprocs=world, join=True)
    for r in range(world):
        failed, opened, err = open(out + f".{r}").read().split(" ", 2)
        assert failed == str(bool(bad))
        assert opened == str(not bad)
        if bad and r not in bad:
            assert "another rank" in err
