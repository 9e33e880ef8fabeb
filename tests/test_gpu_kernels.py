"""GPU kernel-level parity through the C ABI: bit-exact node arithmetic,
deterministic and batch-invariant transforms, device divergence detection,
larger truncations."""

import os

import numpy as np
import pytest

from oracle import sdc as osdc
from oracle.sphere_swe import SphericalShallowWaterOracle, relative_l2
from paper_2403_20135_b200 import (
    CollocationTable,
    DiagonalSdcStepper,
    SdcConfig,
    SerialSdcStepper,
    SweepMode,
    integrate,
    random_initial_state,
)
from paper_2403_20135_b200.errors import DivergenceError
from plan_env import plan_env

pytestmark = pytest.mark.gpu

_P = {}


def gpu(trunc, max_batch=8):
    key = (trunc, max_batch)
    if key not in _P:
        from paper_2403_20135_b200.problem import SphericalShallowWater

        _P[key] = SphericalShallowWater(trunc, max_batch=max_batch)
    return _P[key]


def oracle_for(p, same_tables=False):
    key = ("oracle", p.trunc, same_tables)
    if key not in _P:
        g = p.grid
        tables = None
        if same_tables:
            from paper_2403_20135_b200.sphere import gaussian_latitudes, legendre_tables

            mu, w = gaussian_latitudes(g.nlat)
            pt, ht = legendre_tables(g.trunc, mu)
            tables = (mu, w, pt, ht, p.m_of, p.n_of)
        _P[key] = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon, tables=tables)
    return _P[key]


def test_sweep_nodes_and_final_node_bit_exact():
    """sdcsw_sweep_nodes / sdcsw_final_node == oracle diag_rhs + solve + f_impl, bitwise."""
    import torch

    from paper_2403_20135_b200.integrators import diagonal_step_coefficients
    from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend

    p = gpu(63)
    o = oracle_for(p)
    rng = np.random.default_rng(0)
    m_count, k_count, dt = 4, 3, 90.0
    S = p.state_size
    cfg = SdcConfig(table=CollocationTable.radau_right(m_count), n_sweeps=k_count,
                    mode=SweepMode.DIAGONAL_SEQUENTIAL)
    coef = diagonal_step_coefficients(cfg, dt, p.mean_geopotential)
    blk = m_count * (m_count + 4)
    u0 = rng.standard_normal(S) + 1j * rng.standard_normal(S)
    fe = rng.standard_normal((m_count, S)) + 1j * rng.standard_normal((m_count, S))
    fi = rng.standard_normal((m_count, S)) + 1j * rng.standard_normal((m_count, S))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(p.device)  # noqa: E731
    be = CudaNodeBackend(p)
    u_out = p.empty_states(m_count)
    fi_out = p.empty_states(m_count)
    c1 = np.ascontiguousarray(coef[blk : 2 * blk])  # sweep index 2
    be.sweep_nodes(m_count, 0, m_count, c1, dev(u0), dev(fe), 1, dev(fi), 1, False, u_out, fi_out)
    slots = osdc.Slots(u0, fe[0], fi[0], m_count)
    slots.fe = [fe[j] for j in range(m_count)]
    slots.fi = [fi[j] for j in range(m_count)]
    from paper_2403_20135_b200.collocation import DiagonalPreconditioner, diagonal_coefficients

    table = cfg.table
    diag = diagonal_coefficients(DiagonalPreconditioner.MIN_SR_FLEX, table, 2)
    osdc.diag_rhs(slots, table.q_matrix, dt, diag)
    for m in range(m_count):
        ref_u = o.implicit_solve(dt * diag[m], slots.fi[m])
        assert np.array_equal(u_out[m].cpu().numpy(), ref_u)
        assert np.array_equal(fi_out[m].cpu().numpy(), o.f_impl(ref_u))
    # final node (sweep index K) and the first-sweep aliasing (stride 0, inline f_I(u0))
    out = p.empty_states(1)
    fin = np.ascontiguousarray(coef[(k_count - 1) * blk :])
    be.final_node(m_count, fin, dev(u0), dev(fe), 1, dev(fi), 1, False, out)
    slots = osdc.Slots(u0, fe[0], fi[0], m_count)
    slots.fe = [fe[j] for j in range(m_count)]
    slots.fi = [fi[j] for j in range(m_count)]
    diag = diagonal_coefficients(DiagonalPreconditioner.MIN_SR_FLEX, table, k_count)
    ref = o.implicit_solve(dt * diag[-1], osdc.final_rhs(slots, table.q_matrix, dt, diag))
    assert np.array_equal(out[0].cpu().numpy(), ref)
    be.sweep_nodes(m_count, 1, 2, np.ascontiguousarray(coef[:blk]), dev(u0), dev(fe[0]), 0,
                   dev(fi), 0, True, u_out, fi_out)
    slots = osdc.Slots(u0, fe[0], o.f_impl(u0), m_count)
    diag = diagonal_coefficients(DiagonalPreconditioner.MIN_SR_FLEX, table, 1)
    osdc.diag_rhs(slots, table.q_matrix, dt, diag)
    for q, m in enumerate((1, 2)):
        assert np.array_equal(u_out[q].cpu().numpy(), o.implicit_solve(dt * diag[m], slots.fi[m]))


def test_sweep_nodes_residual_fused():
    """sdcsw_sweep_nodes_residual: the node updates of sdcsw_sweep_nodes (bitwise) plus the
    fused collocation-residual norms ||u0 + sum_j w_mj (fe_j + fi_j) - u_prev_m||_2 per
    (node, field), vs numpy; deterministic across calls; node sub-blocks; first sweep."""
    import torch

    from paper_2403_20135_b200.integrators import diagonal_step_coefficients
    from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend

    p = gpu(127)
    rng = np.random.default_rng(5)
    m_count, dt = 4, 90.0
    S, C = p.state_size, p.n_coef
    cfg = SdcConfig(table=CollocationTable.radau_right(m_count), n_sweeps=3,
                    mode=SweepMode.DIAGONAL_SEQUENTIAL)
    coef = diagonal_step_coefficients(cfg, dt, p.mean_geopotential)
    blk = m_count * (m_count + 4)
    c1 = np.ascontiguousarray(coef[blk : 2 * blk])
    w = c1.reshape(m_count, m_count + 4)
    cplx = lambda *sh: rng.standard_normal(sh) + 1j * rng.standard_normal(sh)  # noqa: E731
    u0, fe, fi = cplx(S), cplx(m_count, S), cplx(m_count, S)
    u_prev = cplx(m_count, S)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(p.device)  # noqa: E731
    be = CudaNodeBackend(p)
    for lo, cnt, first in ((0, m_count, False), (1, 2, False), (0, m_count, True)):
        ua, fa = p.empty_states(cnt), p.empty_states(cnt)
        be.sweep_nodes(m_count, lo, cnt, c1, dev(u0), dev(fe), 1, dev(fi), 1, first, ua, fa)
        res = []
        for _ in range(2):
            ub, fb = p.empty_states(cnt), p.empty_states(cnt)
            r = torch.zeros((cnt, 3), dtype=torch.float64, device=p.device)
            be.sweep_nodes_residual(m_count, lo, cnt, c1, dev(u0), dev(fe), 1, dev(fi), 1, first,
                                    dev(u_prev[lo : lo + cnt]), ub, fb, r)
            assert torch.equal(ua, ub) and torch.equal(fa, fb)
            res.append(r.cpu().numpy())
        assert np.array_equal(res[0], res[1])  # fixed reduction order
        fi_used = np.stack([p.f_impl(u0)] * m_count) if first else fi
        for q in range(cnt):
            m = lo + q
            qf = u0.copy()
            for j in range(m_count):
                qf = qf + w[m, j] * (fe[j] + fi_used[j])
            d = qf - u_prev[m]
            ref = [np.linalg.norm(d[f * C : (f + 1) * C]) for f in range(3)]
            np.testing.assert_allclose(res[0][q], ref, rtol=1e-12)


def test_transforms_deterministic_and_batch_invariant():
    import torch

    p = gpu(127)
    states = np.stack([random_initial_state(p.grid, s) for s in range(6)])
    states[:, : p.n_coef] = 3e-3 * states[:, p.n_coef : 2 * p.n_coef] * 1e6
    u = torch.from_numpy(states).to(p.device)
    outs = []
    for nb in (6, 6, 4, 1):
        o = p.empty_states(6)
        if nb == 6:
            p.f_expl_device(u, o, 6)
        elif nb == 4:
            p.f_expl_device(u[:4].contiguous(), o[:4], 4)
            p.f_expl_device(u[4:].contiguous(), o[4:], 2)
        else:
            for b in range(6):
                p.f_expl_device(u[b : b + 1].contiguous(), o[b : b + 1], 1)
        outs.append(o.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])  # run-to-run deterministic
    assert np.array_equal(outs[0], outs[2])  # independent of the batch split
    assert np.array_equal(outs[0], outs[3])


@pytest.mark.parametrize("trunc,tol", [(255, 1e-11)])
def test_f_expl_large_truncation(trunc, tol):
    p = gpu(trunc, max_batch=4)
    o = oracle_for(p)
    u = random_initial_state(p.grid, 2)
    u[: p.n_coef] = 5e-3 * u[p.n_coef : 2 * p.n_coef] * 1e6
    assert max(relative_l2(p.f_expl(u), o.f_expl(u), o)) < tol


def test_t511_properties():
    """T511 (config 3 size): size-independent checks - exact mass conservation,
    finiteness, f_E linear in Phi' where it should be, solve contract."""
    import torch

    from _contracts import assert_implicit_solve_contract

    p = gpu(511, max_batch=5)
    u0 = random_initial_state(p.grid, 3)
    cfg = SdcConfig(table=CollocationTable.radau_right(5), n_sweeps=5,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=5)
    traj = integrate(p, u0, 30.0, 3, DiagonalSdcStepper(cfg))
    u = traj.states[-1]
    assert np.isfinite(u).all()
    assert u[0] == 0.0  # mean geopotential anomaly: exactly conserved (H_00 = 0)
    assert u[p.n_coef] == 0.0 and u[2 * p.n_coef] == 0.0
    beta = u.copy()
    beta[: p.n_coef] += 1e2 * u[p.n_coef : 2 * p.n_coef] * 1e4
    assert_implicit_solve_contract(p, beta)
    cfg.close()
    del torch


def test_config1_parity_20_steps():
    """BASELINE config 1 (T127, M=4, K=4, dt=90 s) on one GPU, 20 steps, <= 1e-10."""
    p = gpu(127)
    o = oracle_for(p)
    u0 = random_initial_state(p.grid, 1)
    table = CollocationTable.radau_right(4)
    cfg = SdcConfig(table=table, n_sweeps=4, mode=SweepMode.DIAGONAL_PARALLEL, time_threads=4)
    traj = integrate(p, u0, 90.0, 20, DiagonalSdcStepper(cfg), checkpoint_interval=10)
    ref = u0
    for _ in range(20):
        ref = osdc.dsdc(o, ref, 90.0, table, 4)
    assert max(relative_l2(traj.states[-1], ref, o)) <= 1e-10
    assert traj.times == [0.0, 900.0, 1800.0]
    assert [r.n_solve for r in traj.reports] == [13] * 20
    cfg.close()


def test_serial_sdc_parity_10_steps():
    p = gpu(63)
    o = oracle_for(p)
    u0 = random_initial_state(p.grid, 4)
    table = CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.SERIAL)
    traj = integrate(p, u0, 120.0, 10, SerialSdcStepper(cfg))
    ref = u0
    for _ in range(10):
        ref = osdc.serial_sdc(o, ref, 120.0, table, 3)
    assert max(relative_l2(traj.states[-1], ref, o)) <= 1e-10
    cfg.close()


def test_device_divergence_reports_step():
    p = gpu(63)
    u0 = random_initial_state(p.grid, 0) * 1e140  # overflows within the first steps
    table = CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_SEQUENTIAL)
    o = oracle_for(p)
    step = lambda pr, s, dt: osdc.dsdc(pr, s, dt, table, 3)  # noqa: E731
    with pytest.raises(DivergenceError) as ref:
        osdc.march(o, u0, 120.0, 6, step)
    with pytest.raises(DivergenceError) as got:
        integrate(p, u0, 120.0, 6, DiagonalSdcStepper(cfg), checkpoint_interval=6)
    assert got.value.step_index == ref.value.step_index
    cfg.close()


def test_node_parallel_single_rank_matches_fused_stepper():
    """The multi-GPU orchestration at world size 1 over the C-ABI NCCL transport
    (sdcsw_comm_create + sdcsw_allgather_rhs; no torch.distributed at all)
    equals the fused stepper bitwise, eagerly and replayed as one CUDA graph
    with the NCCL all-gathers inside."""
    import torch

    from paper_2403_20135_b200 import _native
    from paper_2403_20135_b200.comm import NcclComm
    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend, NodeParallelDsdc

    assert _native.lib().sdcsw_nccl_version() >= 22700
    p = gpu(63)
    table = CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL, time_threads=1)
    u0 = torch.from_numpy(random_initial_state(p.grid, 8)).to(p.device)
    a = u0.clone()
    npd = NodeParallelDsdc(CudaNodeBackend(p), cfg, 120.0, p.mean_geopotential, p.state_size)
    assert isinstance(npd.node_comm, NcclComm) and npd.node_comm.world == 1
    for _ in range(3):
        npd.step(a)
    b = u0.clone()
    st = DeviceStepper(p, cfg, 120.0, serial=False)
    st.run(b, 3)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    # the same steps captured in one CUDA graph (kernels + NCCL all-gathers)
    c = u0.clone()
    graph = npd.capture(c, 3)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(c, b)
    st.close()
    npd.close()


@pytest.mark.parametrize("trunc,m_count,k_count", [(63, 1, 1), (63, 2, 3), (63, 3, 1), (63, 4, 4),
                                                   (63, 5, 2), (63, 6, 3), (127, 4, 3)])
def test_fused_node_epilogue_bitwise(trunc, m_count, k_count):
    """Node updates fused into the analysis epilogue == separate node kernels
    (batched, chained and sequential), bitwise; launches per step 3K vs 4+4(K-1)."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper

    p = gpu(trunc)
    cfg = SdcConfig(table=CollocationTable.radau_right(m_count), n_sweeps=k_count,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=m_count)
    u0 = torch.from_numpy(random_initial_state(p.grid, 30 + m_count)).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, 90.0, serial=False)
    st.set_chains(1)
    st.set_fused(True)
    assert st.launches_per_step == 3 * k_count
    results = []
    for setup in ("fused", "batched", "chains", "sequential"):
        if setup == "batched":
            st.set_fused(False)
            assert st.launches_per_step == 4 + 4 * (k_count - 1)
        elif setup == "chains":
            st.set_chains(m_count)
        elif setup == "sequential":
            st.set_chains(1)
            st.set_sequential(True)
        u = u0.clone()
        st.run(u, 4)
        torch.cuda.synchronize()
        results.append(u)
    for r in results[1:]:
        assert torch.equal(results[0], r)
    assert st.diverged() == 0
    st.close()


def test_fused_path_divergence_step():
    """The fused closing solve raises the device divergence flag with the step index."""
    from paper_2403_20135_b200.integrators import DeviceStepper

    p = gpu(63)
    table = CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL, time_threads=3)
    u0 = random_initial_state(p.grid, 0) * 1e140
    o = oracle_for(p)
    step = lambda pr, s, dt: osdc.dsdc(pr, s, dt, table, 3)  # noqa: E731
    with pytest.raises(DivergenceError) as ref:
        osdc.march(o, u0, 120.0, 6, step)
    st = DeviceStepper(p, cfg, 120.0, serial=False)
    st.set_chains(1)
    st.set_fused(True)
    u = p._to_device(u0).reshape(-1).contiguous()
    st.run(u, 6)
    assert st.diverged() == ref.value.step_index
    st.close()


def test_ensemble_members_match_single_runs():
    """BASELINE config 4 mechanism: members batched through the GEMMs give, per
    member, exactly the single-state result (bitwise)."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper

    p = gpu(63, max_batch=12)
    table = CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL, time_threads=3)
    states = np.stack([random_initial_state(p.grid, 20 + e) for e in range(4)])
    ens = torch.from_numpy(states).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, 120.0, serial=False, members=4)
    st.run(ens, 3)
    single = DeviceStepper(p, cfg, 120.0, serial=False)
    for e in range(4):
        u = torch.from_numpy(states[e]).to(p.device).contiguous()
        single.run(u, 3)
        assert torch.equal(u, ens[e])
    assert st.diverged() == 0
    st.close()
    single.close()


@pytest.mark.parametrize("trunc,nparts", [(127, 2), (127, 4), (255, 2), (255, 3)])
def test_spectral_split_f_expl_bitwise(trunc, nparts):
    """Spectral split kernels on one device: the parts are run one
    after another into a shared part-major Fourier buffer (no inter-rank
    waiting), and the own-m tendencies they produce, combined, equal the
    unsplit f_E bit for bit."""
    import torch

    from paper_2403_20135_b200 import _native
    from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend, spectral_parts
    from paper_2403_20135_b200.problem import SphericalShallowWater

    p = SphericalShallowWater(trunc, max_batch=2)
    nb = 2
    states = np.stack([random_initial_state(p.grid, 40 + b) for b in range(nb)])
    states[:, : p.n_coef] = 2e-3 * states[:, p.n_coef : 2 * p.n_coef] * 1e6
    u = torch.from_numpy(states).to(p.device).contiguous()
    ref = p.empty_states(nb)
    p.f_expl_device(u, ref, nb)
    be = CudaNodeBackend(p)
    be.set_split(nparts, 0, nb)
    got = torch.zeros_like(ref)
    outs = []
    for q in range(nparts):  # all synthesis parts first (the all-gather's effect)
        _native.check(p._lib.sdcsw_plan_set_split(p.handle, nparts, q, be.fourier.data_ptr(),
                                                  be.fourier.numel() * 16))
        _native.check(p._lib.sdcsw_split_f_expl_begin(p.handle, u.data_ptr(), nb, p.stream()))
    for q in range(nparts):
        # re-select part q without clearing the shared Fourier buffer
        _native.check(p._lib.sdcsw_plan_set_split(p.handle, nparts, q, be.fourier.data_ptr(),
                                                  be.fourier.numel() * 16))
        o = torch.zeros_like(ref)
        _native.check(p._lib.sdcsw_split_f_expl_end(p.handle, o.data_ptr(), nb, p.stream()))
        outs.append(o)
    part_of = np.array(spectral_parts(trunc, nparts))
    for q in range(nparts):
        own = torch.from_numpy(np.tile(part_of[p.m_of] == q, 3)).to(p.device)
        got[:, own] = outs[q][:, own]
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    _native.check(p._lib.sdcsw_plan_set_split(p.handle, 1, 0, None, 0))
    p.close()


def test_reference_schemes_on_gpu():
    """IMEX-o2 / AB2-SI on the device problem vs the oracle restatement (pinned to the reference)."""
    from paper_2403_20135_b200.schemes import Ab2SiStepper, ImexO2Stepper

    p = gpu(63)
    o = oracle_for(p)
    u0 = random_initial_state(p.grid, 6)
    traj = integrate(p, u0, 120.0, 5, ImexO2Stepper())
    ref = u0
    for _ in range(5):
        ref = osdc.imex_o2(o, ref, 120.0)
    assert max(relative_l2(traj.states[-1], ref, o)) <= 1e-10
    assert [(r.n_f_expl, r.n_f_impl, r.n_solve) for r in traj.reports] == [(2, 2, 2)] * 5
    traj = integrate(p, u0, 120.0, 5, Ab2SiStepper())
    assert max(relative_l2(traj.states[-1], osdc.ab2_run(o, u0, 120.0, 5), o)) <= 1e-10
    assert [(r.n_f_expl, r.n_f_impl, r.n_solve) for r in traj.reports] == [(3, 2, 2)] + [(1, 1, 1)] * 4


def test_tma_analysis_matches_latency_analysis_t511():
    """T511: the table-streaming TMA analysis (fragment-order analysis data) and
    the latency-regime analysis (record order; forced with SDCSW_ANAL_WJ=2) give
    the same f_E to summation-order rounding (both with the P/H tables: the H-free
    path is compared in test_ponly_matches_ph_and_oracle)."""
    from paper_2403_20135_b200.problem import SphericalShallowWater

    with plan_env(SDCSW_PONLY="0"):
        p = SphericalShallowWater(511, max_batch=5)
    u = random_initial_state(p.grid, 11)
    u[: p.n_coef] = 4e-3 * u[p.n_coef : 2 * p.n_coef] * 1e6
    a = p.f_expl(u)
    with plan_env(SDCSW_ANAL_WJ="2"):
        q = SphericalShallowWater(511, max_batch=2)
    b = q.f_expl(u)
    c = p.n_coef
    for f in range(3):
        x, y = a[f * c : (f + 1) * c], b[f * c : (f + 1) * c]
        assert np.linalg.norm(x - y) <= 1e-12 * np.linalg.norm(y)
    q.close()
    p.close()


@pytest.mark.parametrize("trunc,max_batch,nb", [(255, 4, 4), (511, 5, 5), (127, 16, 16)])
def test_ponly_matches_ph_and_oracle(trunc, max_batch, nb):
    """H-free transforms (legendre_ponly.cu: P tables to degree T+1, the derivative
    recurrence for H) against the P/H path on the same plan shape and against the CPU
    oracle with its own (independent) tables: f_E agrees with the P/H path to 3e-12
    relative per field and state, and its error against the oracle is no larger than
    the P/H path's (within a factor 2, floor 1e-12)."""
    import torch

    from paper_2403_20135_b200.problem import SphericalShallowWater

    with plan_env(SDCSW_PONLY="1"):
        po = SphericalShallowWater(trunc, max_batch=max_batch)
    with plan_env(SDCSW_PONLY="0"):
        ph = SphericalShallowWater(trunc, max_batch=max_batch)
    assert po.uses_ponly and not ph.uses_ponly
    c = po.n_coef
    states = np.stack([random_initial_state(po.grid, 90 + b) for b in range(nb)])
    states[:, :c] = 4e-3 * states[:, c : 2 * c] * 1e6
    u = torch.from_numpy(states).to(po.device).contiguous()
    a = po.f_expl_device(u, po.empty_states(nb), nb).cpu().numpy()
    b = ph.f_expl_device(u, ph.empty_states(nb), nb).cpu().numpy()
    for s in range(nb):
        for f in range(3):
            x, y = a[s, f * c : (f + 1) * c], b[s, f * c : (f + 1) * c]
            assert np.linalg.norm(x - y) <= 3e-12 * np.linalg.norm(y), (s, f)
    o = oracle_for(po)
    for s in (0, nb - 1):
        ref = o.f_expl(states[s])
        e_po = max(relative_l2(a[s], ref, o))
        e_ph = max(relative_l2(b[s], ref, o))
        assert e_po <= max(2 * e_ph, 1e-12), (e_po, e_ph)
    po.close()
    ph.close()


def test_plans_of_different_sizes_coexist():
    """Kernel attributes are process-wide: creating a small plan after a large
    one must not break the large one (ring shared-memory limits)."""
    from paper_2403_20135_b200.problem import SphericalShallowWater

    big = gpu(511, max_batch=5)
    u = random_initial_state(big.grid, 12)
    a = big.f_expl(u)
    small = SphericalShallowWater(63, max_batch=2)
    small.f_expl(random_initial_state(small.grid, 1))
    assert np.array_equal(big.f_expl(u), a)
    small.close()


def test_graph_steps_bitwise():
    """Several steps per replayed graph (PDL across step boundaries) == one step
    per graph == eager launches, bitwise, including a remainder."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper

    p = gpu(63)
    cfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=3,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=3)
    u0 = torch.from_numpy(random_initial_state(p.grid, 40)).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, 120.0, serial=False)
    out = []
    for g, graph in ((1, True), (8, True), (5, True), (1, False)):
        st.set_graph_steps(g)
        u = u0.clone()
        st.run(u, 11, use_graph=graph)
        torch.cuda.synchronize()
        out.append(u)
    for o in out[1:]:
        assert torch.equal(out[0], o)
    st.close()


def test_throughput_regime_batch_consistent():
    """Large batches (ensemble-size: the GEMMs' throughput regime, no K-split,
    several batch blocks per CTA, cp.async synthesis) agree with the single-state
    f_E to summation-order rounding, and are bitwise reproducible run to run."""
    import torch

    p = gpu(63, max_batch=40)
    o = oracle_for(p)
    states = np.stack([random_initial_state(p.grid, 50 + b) for b in range(40)])
    u = torch.from_numpy(states).to(p.device).contiguous()
    big, again = p.empty_states(40), p.empty_states(40)
    p.f_expl_device(u, big, 40)
    p.f_expl_device(u, again, 40)
    assert torch.equal(big, again)
    for b in (0, 7, 21, 39):
        one = p.empty_states(1)
        p.f_expl_device(u[b : b + 1].contiguous(), one, 1)
        assert max(relative_l2(big[b].cpu().numpy(), one[0].cpu().numpy(), o)) < 1e-13


@pytest.mark.parametrize("trunc,m_count,k_count", [(63, 3, 3), (63, 1, 2), (127, 4, 4), (63, 5, 1)])
def test_serial_fused_epilogue_bitwise(trunc, m_count, k_count):
    """Serial SDC with serial_update / serial_node in the analysis epilogue ==
    the separate serial kernels, bitwise (divergence flag untouched)."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper

    p = gpu(trunc)
    cfg = SdcConfig(table=CollocationTable.radau_right(m_count), n_sweeps=k_count,
                    mode=SweepMode.SERIAL)
    u0 = torch.from_numpy(random_initial_state(p.grid, 60 + m_count)).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, 90.0, serial=True)
    st.set_fused(True)
    assert st.launches_per_step == 3 + k_count * (2 + 3 * m_count)
    a = u0.clone()
    st.run(a, 3)
    st.set_fused(False)
    assert st.launches_per_step == 3 + k_count * 5 * m_count
    b = u0.clone()
    st.run(b, 3)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert st.diverged() == 0
    st.close()


def test_serial_divergence_reports_step():
    p = gpu(63)
    u0 = random_initial_state(p.grid, 0) * 1e140
    table = CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.SERIAL)
    o = oracle_for(p)
    step = lambda pr, s, dt: osdc.serial_sdc(pr, s, dt, table, 3)  # noqa: E731
    with pytest.raises(DivergenceError) as ref:
        osdc.march(o, u0, 120.0, 6, step)
    with pytest.raises(DivergenceError) as got:
        integrate(p, u0, 120.0, 6, SerialSdcStepper(cfg), checkpoint_interval=6)
    assert got.value.step_index == ref.value.step_index
    cfg.close()


@pytest.mark.parametrize("nb,max_batch", [(8, 8), (8, 12), (25, 25), (13, 18)])
def test_bulk_synthesis_partial_batch_block(nb, max_batch):
    """Bulk-staged synthesis with nb > 6 states (batch blocks of 6 along grid z,
    the last one partial): every state's Fourier coefficients are
    bitwise equal to a one-state synthesis of it (per-column sums do not depend
    on the batch), agree with the cp.async synthesis to rounding, and the
    workspace entries of states nb..max_batch-1 keep a sentinel (no store past
    the last state)."""
    import torch

    from paper_2403_20135_b200.problem import SphericalShallowWater

    def plan(bulk):
        # P/H tables (ensemble plans from 16 states would take the H-free path,
        # whose synthesis is always the bulk kernel: test_ponly_partial_batch_block)
        with plan_env(SDCSW_SYN_BULK=bulk, SDCSW_PONLY="0"):
            return SphericalShallowWater(127, max_batch=max_batch)

    def synth(p, u, nb):
        s = p.stream()
        _native_check(p, 0, u, nb, s)
        _native_check(p, 3, u, nb, s)
        torch.cuda.synchronize()
        return p.workspace(0).view(max_batch, -1)

    pb, pc = plan("1"), plan("0")
    states = np.stack([random_initial_state(pb.grid, 70 + b) for b in range(nb)])
    u = torch.from_numpy(states).to(pb.device).contiguous()
    wb = pb.workspace(0).view(max_batch, -1)
    wb.fill_(12345.0)
    bulk = synth(pb, u, nb).clone()
    assert torch.isfinite(bulk[:nb]).all()
    assert (bulk[nb:] == 12345.0).all()
    cp = synth(pc, u, nb).clone()
    d = (bulk[:nb] - cp[:nb]).abs().max().item()
    assert d <= 1e-13 * cp[:nb].abs().max().item()
    for b in sorted({0, 5, 6, nb - 2, nb - 1}):
        one = synth(pb, u[b : b + 1].contiguous(), 1)
        assert torch.equal(one[0], bulk[b]), b
    pb.close()
    pc.close()


@pytest.mark.parametrize("nb,max_batch", [(25, 25), (13, 18), (8, 16)])
def test_ponly_partial_batch_block(nb, max_batch):
    """H-free synthesis (operand conversion + P-only bulk kernel) with batch blocks of
    6 states, the last one partial: every state's Fourier coefficients are bitwise
    those of a one-state synthesis, and the workspace entries of states
    nb..max_batch-1 keep a sentinel (no store past the last state)."""
    import torch

    from paper_2403_20135_b200.problem import SphericalShallowWater

    with plan_env(SDCSW_PONLY="1"):
        p = SphericalShallowWater(127, max_batch=max_batch)
    assert p.uses_ponly
    states = np.stack([random_initial_state(p.grid, 170 + b) for b in range(nb)])
    u = torch.from_numpy(states).to(p.device).contiguous()
    w = p.workspace(0).view(max_batch, -1)
    w.fill_(12345.0)

    def synth(x, n):
        _native_check(p, 0, x, n, p.stream())
        torch.cuda.synchronize()
        return w.clone()

    full = synth(u, nb)
    assert torch.isfinite(full[:nb]).all()
    assert (full[nb:] == 12345.0).all()
    for b in sorted({0, 5, 6, nb - 2, nb - 1}):
        one = synth(u[b : b + 1].contiguous(), 1)
        assert torch.equal(one[0], full[b]), b
    p.close()


def _native_check(p, stage, u, nb, s):
    from paper_2403_20135_b200 import _native

    out = p.empty_states(nb)
    _native.check(p._lib.sdcsw_transform_stage(p.handle, stage, u.data_ptr(), out.data_ptr(), nb, s))


def test_on_sweep_callback_and_storage_accounting():
    """dsdc_step / sdc_step_serial accept the reference's on_sweep(k, state)
    callback (integrators.py:317-381): called after every sweep with the sweep
    storage; the step result is bitwise that of the fused step; the retained
    arrays stay within the reference's 2M + 3 bound
    (pkg/tests/test_integrators.py:228-241) and the counts are (13, 13, 13)
    for M = K = 4 (criterion 7, pkg/tests/test_acceptance.py:284-305).  The
    stepper's allocated sweep storage is 1 + 4M state buffers."""
    from paper_2403_20135_b200 import dsdc_step, sdc_step_serial
    from paper_2403_20135_b200.core import evaluation_counters
    from paper_2403_20135_b200.integrators import _device_stepper

    p = gpu(63)
    u0 = random_initial_state(p.grid, 21)
    cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=4, mode=SweepMode.DIAGONAL_SEQUENTIAL)
    plain, _ = dsdc_step(p, u0, 120.0, cfg)
    seen = []

    def cb(k, state):
        seen.append((k, state.distinct_node_arrays(), state.fe0.copy(), state.fe, state.fi, state.u))

    before = evaluation_counters(p)
    hooked, rep = dsdc_step(p, u0, 120.0, cfg, on_sweep=cb)
    after = evaluation_counters(p)
    assert np.array_equal(hooked, plain)
    assert tuple(a - b for a, b in zip(after, before)) == (13, 13, 13)
    assert [s[0] for s in seen] == [1, 2, 3]
    assert all(s[1] <= 2 * 4 + 3 for s in seen)
    assert all(len(s[3]) == 4 and len(s[4]) == 4 and s[5] == [None] * 4 for s in seen)
    # fe0 is f_E(u0); the tendencies change from sweep to sweep
    fe0_ref = p.f_expl(u0)
    assert max(relative_l2(seen[0][2], fe0_ref, oracle_for(p))) < 1e-14
    assert not np.array_equal(seen[0][3][1], seen[1][3][1])
    assert rep.init_s > 0 and len(rep.sweep_s) == 3 and rep.final_node_s > 0
    st = _device_stepper(cfg, p, 120.0, False)
    nbytes, nbuf = st.storage()
    assert nbuf == 1 + 4 * 4 and nbytes >= nbuf * p.state_size * 16
    scfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=2, mode=SweepMode.SERIAL)
    ks = []
    out_s, _ = sdc_step_serial(p, u0, 120.0, scfg, on_sweep=lambda k, s: ks.append(k))
    assert ks == [1, 2]
    assert np.array_equal(out_s, sdc_step_serial(p, u0, 120.0, scfg)[0])
    cfg.close()
    scfg.close()


def test_integrate_stage_timings_feed_the_perf_model():
    """integrate(..., stage_timings=True) fills init_s / sweep_s / final_node_s
    of every StepReport from CUDA events (bitwise the same states), so the
    reference's perfmodel.fit_costs (pkg/src/parsdc/perfmodel.py:78-111) runs on
    a normal integrate() call."""
    from paper_2403_20135_b200.perfmodel import fit_costs

    p = gpu(63)
    u0 = random_initial_state(p.grid, 22)
    # sequential node updates (the reference's DIAGONAL_SEQUENTIAL): the cost
    # model's per-node structure (the batched parallel sweep costs about one node)
    cfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=3, mode=SweepMode.DIAGONAL_SEQUENTIAL)
    fast = integrate(p, u0, 120.0, 6, DiagonalSdcStepper(cfg), checkpoint_interval=3)
    timed = integrate(p, u0, 120.0, 6, DiagonalSdcStepper(cfg), checkpoint_interval=3, stage_timings=True)
    for a, b in zip(fast.states, timed.states):
        assert np.array_equal(a, b)
    assert len(timed.reports) == 6
    assert all(r.init_s > 0 and len(r.sweep_s) == 2 and min(r.sweep_s) > 0 and r.final_node_s > 0
               for r in timed.reports)
    model = fit_costs(timed.reports, 3)
    assert model.c_e > 0
    cfg.close()


@pytest.mark.parametrize("trunc,m_count,k_count", [(63, 3, 3), (127, 4, 2)])
def test_standalone_serial_sweep_matches_serial_step(trunc, m_count, k_count):
    """sdcsw_serial_sweep (the reference's serial_sweep, integrators.py:183-230):
    f_E(u0) followed by K standalone serial sweeps reproduces the serial SDC
    stepper's step bitwise (SURVEY 8(b) sdcsw_serial_sweep)."""
    import torch

    from paper_2403_20135_b200 import sdc_step_serial
    from paper_2403_20135_b200.integrators import serial_step_coefficients
    from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend

    p = gpu(trunc)
    cfg = SdcConfig(table=CollocationTable.radau_right(m_count), n_sweeps=k_count, mode=SweepMode.SERIAL)
    u0 = random_initial_state(p.grid, 31)
    want, _ = sdc_step_serial(p, u0, 100.0, cfg)
    coef = np.ascontiguousarray(serial_step_coefficients(cfg, 100.0, p.mean_geopotential,
                                                         p.solve_coefficients))
    b = CudaNodeBackend(p)
    u = torch.from_numpy(u0).to(p.device).reshape(1, -1).contiguous()
    fe0 = p.empty_states(1)
    p.f_expl_device(u, fe0, 1)
    fe = [p.empty_states(m_count) for _ in range(2)]
    fi = [p.empty_states(m_count) for _ in range(2)]
    last, work = p.empty_states(1), p.empty_states(m_count + 2)
    old_fe, old_fi, stride, first = fe0, fe0, 0, True
    for k in range(k_count):
        b.serial_sweep(m_count, coef, u, old_fe, stride, old_fi, stride, first, fe[k % 2], fi[k % 2],
                       last, work)
        old_fe, old_fi, stride, first = fe[k % 2], fi[k % 2], 1, False
    torch.cuda.synchronize()
    assert np.array_equal(last[0].cpu().numpy(), want)
    cfg.close()


def test_nccl_allgather_through_the_c_abi():
    """sdcsw_comm_init_all / sdcsw_comm_create + sdcsw_allgather_rhs on one GPU:
    the all-gather of one rank is a copy, in place and out of place."""
    import torch

    from paper_2403_20135_b200.comm import NcclComm

    comms = NcclComm.init_all([0])
    assert len(comms) == 1 and comms[0].world == 1 and comms[0].rank == 0
    boot = NcclComm.create(NcclComm.unique_id(), 1, 0, 0)
    x = torch.randn(1000, dtype=torch.float64, device="cuda")
    for c in (comms[0], boot):
        y = torch.zeros_like(x)
        c.allgather(y, x, ctypes_stream())
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        z = x.clone()
        c.allgather(z, z, ctypes_stream())  # in place
        torch.cuda.synchronize()
        assert torch.equal(z, x)
        c.close()


def ctypes_stream():
    import ctypes

    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def test_dsdc_order_and_sweep_monotonicity_on_the_sphere():
    """The reference's integrator oracles (pkg/tests/test_integrators.py:270-305)
    run on the device stepper with the spherical problem: M = K = 4 dSDC
    converges with order >= 3.5 in dt (errors against a fine-step run of the
    same scheme over a fixed 2 h horizon), and at fixed dt the error falls
    monotonically with the sweep count K = 1..4."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper

    p = gpu(63)
    u0 = torch.from_numpy(random_initial_state(p.grid, 5)).to(p.device).reshape(-1).contiguous()
    horizon = 7200.0

    def run(n_steps, k):
        cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=k,
                        mode=SweepMode.DIAGONAL_PARALLEL)
        st = DeviceStepper(p, cfg, horizon / n_steps, serial=False)
        u = u0.clone()
        st.run(u, n_steps)
        torch.cuda.synchronize()
        st.close()
        return u.cpu().numpy()

    ref = run(256, 4)
    o = oracle_for(p)
    dts, errs = [], []
    for n in (8, 16, 32, 64):
        dts.append(horizon / n)
        errs.append(max(relative_l2(run(n, 4), ref, o)))
    slope = np.polyfit(np.log(dts), np.log(errs), 1)[0]
    print(f"dSDC M=K=4 order on the sphere: slope {slope:.2f}, errors {errs}")
    assert slope >= 3.5, (slope, errs)
    by_k = [max(relative_l2(run(16, k), ref, o)) for k in range(1, 5)]
    print(f"errors by sweep count K=1..4 at 16 steps: {by_k}")
    assert all(b < a for a, b in zip(by_k, by_k[1:])), by_k


@pytest.mark.parametrize(
    "trunc,grid,nb,max_batch,ponly",
    [(42, (64, 192), 2, 2, None), (85, (128, 384), 3, 3, None), (127, None, 4, 4, None),
     (127, None, 20, 32, None), (127, None, 20, 32, "0"), (383, (576, 1536), 1, 1, None),
     (511, None, 2, 2, None), (511, None, 2, 2, "0")],
)
def test_ring_tma_stores_match_plain_stores(trunc, grid, nb, max_batch, ponly):
    """The ring kernel's analysis data written by TMA tensor stores from shared
    memory (record order; fragment order from T200 and for ensembles; one box
    of L rows - 43 and 86 included - or 192 / 256-row boxes at T383 / T511) is bitwise the data of the
    per-thread stores (SDCSW_RING_TMA_STORE=0): f_E agrees bit for bit.  Table-streaming
    plans (T >= 200, ensembles) run H-free with the five-slot data; ponly = "0" forces
    the P/H tables and the seven-slot fragment order."""
    from paper_2403_20135_b200.problem import SphericalShallowWater

    plans = []
    extra = {"SDCSW_PONLY": ponly} if ponly else {}
    for mode in ("1", "0"):
        with plan_env(SDCSW_RING_TMA_STORE=mode, **extra):
            nlat, nlon = grid or (None, None)
            plans.append(SphericalShallowWater(trunc, nlat=nlat, nlon=nlon, max_batch=max_batch))
    import torch

    g, c = plans[0].grid, plans[0].n_coef
    states = np.stack([random_initial_state(g, 3 + s) for s in range(nb)])
    states[:, :c] = 4e-3 * states[:, c : 2 * c] * 1e6
    outs = []
    for p in plans:
        u = torch.from_numpy(states).to(p.device)
        outs.append(p.f_expl_device(u, p.empty_states(nb), nb).cpu().numpy())
    a, b = outs
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert np.all(np.isfinite(a)) and np.linalg.norm(a) > 0
    for p in plans:
        p.close()


def test_ponly_stepper_ensemble_matches_single_runs():
    """H-free dSDC stepper (operand built from the node states, k_prep_ponly) at T255:
    an ensemble of 2 members gives, per member, exactly the single-member result, and
    both agree with the P/H stepper to rounding."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.problem import SphericalShallowWater

    with plan_env(SDCSW_PONLY="1"):
        p = SphericalShallowWater(255, max_batch=6)
    with plan_env(SDCSW_PONLY="0"):
        q = SphericalShallowWater(255, max_batch=3)
    assert p.uses_ponly and not q.uses_ponly
    cfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=2,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=3)
    states = np.stack([random_initial_state(p.grid, 60 + e) for e in range(2)])
    ens = torch.from_numpy(states).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, 60.0, serial=False, members=2)
    st.run(ens, 2)
    single = DeviceStepper(p, cfg, 60.0, serial=False)
    ref = DeviceStepper(q, cfg, 60.0, serial=False)
    o = oracle_for(p)
    for e in range(2):
        u = torch.from_numpy(states[e]).to(p.device).contiguous()
        single.run(u, 2)
        assert torch.equal(u, ens[e])
        v = torch.from_numpy(states[e]).to(q.device).contiguous()
        ref.run(v, 2)
        assert max(relative_l2(u.cpu().numpy(), v.cpu().numpy(), o)) < 1e-12
    for s in (st, single, ref):
        s.close()
    p.close()
    q.close()


def test_ponly_serial_sdc_matches_ph():
    """Serial SDC on an H-free plan (operand records + conversion route) against the
    P/H tables at T255: two steps agree to rounding."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.problem import SphericalShallowWater

    with plan_env(SDCSW_PONLY="1"):
        p = SphericalShallowWater(255, max_batch=4)
    with plan_env(SDCSW_PONLY="0"):
        q = SphericalShallowWater(255, max_batch=4)
    cfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=2, mode=SweepMode.SERIAL)
    u0 = random_initial_state(p.grid, 66)
    out = []
    for prob in (p, q):
        st = DeviceStepper(prob, cfg, 60.0, serial=True)
        u = torch.from_numpy(u0).to(prob.device).contiguous()
        st.run(u, 2)
        out.append(u.cpu().numpy())
        st.close()
    assert max(relative_l2(out[0], out[1], oracle_for(p))) < 1e-12
    p.close()
    q.close()


def test_ponly_t383_f_expl_vs_oracle():
    """H-free f_E on a non-power-of-two grid (T383, 576 x 1536: L = 384, 192-row TMA store
    boxes) against the CPU oracle with its own tables."""
    from paper_2403_20135_b200.problem import SphericalShallowWater

    p = SphericalShallowWater(383, nlat=576, nlon=1536, max_batch=2)
    assert p.uses_ponly
    u = random_initial_state(p.grid, 77)
    u[: p.n_coef] = 4e-3 * u[p.n_coef : 2 * p.n_coef] * 1e6
    o = SphericalShallowWaterOracle(p.grid.trunc, p.grid.nlat, p.grid.nlon)
    assert max(relative_l2(p.f_expl(u), o.f_expl(u), o)) < 1e-10
    p.close()


@pytest.mark.parametrize("trunc,m_count,k_count,members", [(255, 4, 3, 1), (127, 4, 2, 6)])
def test_ponly_node_kernel_operand_bitwise(trunc, m_count, k_count, members):
    """H-free dSDC: the sweep's node kernel writing the P-only synthesis operand itself
    (k_sweep_nodes_po, neighbour degrees by warp shuffles across a 30 + 2 halo lane
    layout) gives bit for bit the result of storing the node states and building the
    operand from them (k_prep_ponly; SDCSW_NODES_PO=0)."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.problem import SphericalShallowWater

    outs = []
    for po in ("1", "0"):
        with plan_env(SDCSW_NODES_PO=po, SDCSW_PONLY="1"):
            p = SphericalShallowWater(trunc, max_batch=m_count * members)
            cfg = SdcConfig(table=CollocationTable.radau_right(m_count), n_sweeps=k_count,
                            mode=SweepMode.DIAGONAL_PARALLEL)
            st = DeviceStepper(p, cfg, 60.0, serial=False, members=members)
        assert p.uses_ponly
        u0 = np.stack([random_initial_state(p.grid, 15 + e) for e in range(members)])
        u = torch.from_numpy(u0).to(p.device).reshape(-1).contiguous()
        st.run(u, 3)
        torch.cuda.synchronize()
        outs.append(u.cpu().numpy())
        st.close()
        p.close()
    assert np.array_equal(outs[0].view(np.uint64), outs[1].view(np.uint64))


def test_ponly_stepper_chains_and_sequential_bitwise():
    """H-free dSDC at T255 (the node kernel writing the P-only operand into each chain's
    workspace slice): concurrent node chains (2 and 4 graph branches) and sequential node
    updates give the batched result bit for bit."""
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.problem import SphericalShallowWater

    with plan_env(SDCSW_PONLY="1"):
        p = SphericalShallowWater(255, max_batch=4)
    cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=3,
                    mode=SweepMode.DIAGONAL_PARALLEL)
    u0 = torch.from_numpy(random_initial_state(p.grid, 88)).to(p.device).contiguous()
    outs = []
    for chains, seq in ((1, False), (2, False), (4, False), (1, True)):
        st = DeviceStepper(p, cfg, 60.0, serial=False)
        st.set_chains(chains)
        st.set_sequential(seq)
        u = u0.clone()
        st.run(u, 3)
        torch.cuda.synchronize()
        outs.append(u)
        st.close()
    for o in outs[1:]:
        assert torch.equal(outs[0], o)
    p.close()


@pytest.mark.parametrize("trunc,nlat,nlon,max_batch", [(210, 320, 768, 3), (301, 448, 768, 2)])
def test_ponly_odd_sizes_vs_oracle(trunc, nlat, nlon, max_batch):
    """H-free plans of unusual shape - odd L = T + 1 (211-row TMA store boxes), nlat/2 not a
    multiple of 64 (two-warp synthesis CTAs), degree-(T+1) rows of odd and even parity -
    against the CPU oracle with its own tables, for a batch of states."""
    import torch

    from paper_2403_20135_b200.problem import SphericalShallowWater

    p = SphericalShallowWater(trunc, nlat=nlat, nlon=nlon, max_batch=max_batch)
    assert p.uses_ponly
    c = p.n_coef
    states = np.stack([random_initial_state(p.grid, 120 + b) for b in range(max_batch)])
    states[:, :c] = 4e-3 * states[:, c : 2 * c] * 1e6
    u = torch.from_numpy(states).to(p.device).contiguous()
    out = p.f_expl_device(u, p.empty_states(max_batch), max_batch).cpu().numpy()
    o = SphericalShallowWaterOracle(p.grid.trunc, p.grid.nlat, p.grid.nlon)
    for b in (0, max_batch - 1):
        assert max(relative_l2(out[b], o.f_expl(states[b]), o)) < 1e-10
    p.close()
