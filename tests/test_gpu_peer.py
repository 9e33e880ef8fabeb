"""Node-parallel dSDC over peer memory (csrc/peer.cu, sdcsw_exchange_*) on one
B200.

World size 1 runs the full protocol (publish into the exchange buffer, post
the flag, wait, read the parity) against the process's own buffer.  Larger
worlds run as several exchange objects of one process attached to each other,
with the phases of all ranks interleaved on ONE stream and the posts a phase
consumes enqueued for every rank before it (run_in_stream_order): every wait
is already satisfied by kernels earlier in the stream, so no kernel ever waits
on a concurrently running one.  Each rank must end bit-identical to the
single-GPU stepper (the reference's thread-count invariance,
pkg/tests/test_integrators.py:190-225)."""

import pytest

from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state

pytestmark = pytest.mark.gpu

_P = {}


def gpu(trunc, max_batch=8):
    key = (trunc, max_batch)
    if key not in _P:
        from paper_2403_20135_b200.problem import SphericalShallowWater

        _P[key] = SphericalShallowWater(trunc, max_batch=max_batch)
    return _P[key]


def _cfg(m, k):
    return SdcConfig(table=CollocationTable.radau_right(m), n_sweeps=k,
                     mode=SweepMode.DIAGONAL_PARALLEL, time_threads=1)


def _stepper_result(p, cfg, dt, u0, n):
    from paper_2403_20135_b200.integrators import DeviceStepper

    b = u0.clone()
    st = DeviceStepper(p, cfg, dt, serial=False)
    st.run(b, n)
    st.close()
    return b


@pytest.mark.parametrize("trunc,m,k", [(63, 3, 3), (127, 4, 4), (63, 2, 1), (63, 6, 2), (63, 8, 3)])
@pytest.mark.parametrize("fused", [True, False])
def test_exchange_single_rank_bitwise(trunc, m, k, fused):
    import torch

    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

    p = gpu(trunc)
    cfg = _cfg(m, k)
    u0 = torch.from_numpy(random_initial_state(p.grid, 3)).to(p.device)
    ref = _stepper_result(p, cfg, 90.0, u0, 5)
    x = PeerNodeParallelDsdc(p, cfg, 90.0, world=1, rank=0, fused=fused)
    assert x.info()[:2] == (0, m)
    a = u0.clone()
    x.run(a, 5, use_graph=False)
    torch.cuda.synchronize()
    assert torch.equal(a, ref)
    c = u0.clone()
    x.run(c, 2, use_graph=True)   # one-step graph twice
    x.run(c, 3, use_graph=True)
    torch.cuda.synchronize()
    assert torch.equal(c, ref)
    x.close()


@pytest.mark.parametrize("m,world", [(4, 2), (4, 4), (3, 2), (5, 3), (2, 4), (6, 4), (7, 2), (8, 3)])
@pytest.mark.parametrize("fused", [True, False])
def test_exchange_ranks_interleaved_bitwise(m, world, fused):
    import torch

    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc, node_block

    p = gpu(63)
    k = 3
    cfg = _cfg(m, k)
    u0 = torch.from_numpy(random_initial_state(p.grid, 11)).to(p.device)
    n_steps = 4
    ref = _stepper_result(p, cfg, 120.0, u0, n_steps)
    ranks = PeerNodeParallelDsdc.in_process(p, cfg, 120.0, world, fused=fused)
    for x in ranks:
        lo, count, _ = node_block(m, world, x.rank)
        assert x.info()[:2] == (lo, count)
    states = [u0.clone() for _ in ranks]
    PeerNodeParallelDsdc.run_in_stream_order(ranks, states, n_steps)
    torch.cuda.synchronize()
    for u in states:
        assert torch.equal(u, ref)
    for x in ranks:
        assert x.diverged() == 0
        x.close()


def test_exchange_table_streaming_copy_publish():
    """T511 (TMA analysis, no fused epilogue): the copy-kernel publish."""
    import torch

    from paper_2403_20135_b200.errors import ParameterError
    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

    p = gpu(511, max_batch=4)
    cfg = _cfg(3, 2)
    u0 = torch.from_numpy(random_initial_state(p.grid, 5)).to(p.device)
    ref = _stepper_result(p, cfg, 30.0, u0, 2)
    ranks = PeerNodeParallelDsdc.in_process(p, cfg, 30.0, 2)
    with pytest.raises(ParameterError):
        ranks[0].set_fused(True)
    states = [u0.clone() for _ in ranks]
    PeerNodeParallelDsdc.run_in_stream_order(ranks, states, 2)
    torch.cuda.synchronize()
    for u in states:
        assert torch.equal(u, ref)
    for x in ranks:
        x.close()


def test_exchange_divergence_step_index():
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

    p = gpu(63)
    cfg = _cfg(3, 3)
    u0 = torch.from_numpy(random_initial_state(p.grid, 0) * 1e140).to(p.device)
    st = DeviceStepper(p, cfg, 120.0, serial=False)
    b = u0.clone()
    st.run(b, 6)
    want = st.diverged()
    st.close()
    assert want > 0
    x = PeerNodeParallelDsdc(p, cfg, 120.0, world=1, rank=0)
    a = u0.clone()
    x.run(a, 6)
    assert x.diverged() == want
    x.close()


def test_exchange_launch_count():
    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

    p = gpu(127)
    ranks = PeerNodeParallelDsdc.in_process(p, _cfg(4, 4), 90.0, 4)
    # init f_E 3 + 3 sweeps x (node, synthesis, ring, analysis) + closing solve
    assert [x.info()[2] for x in ranks] == [16] * 4
    ranks[0].set_fused(False)
    assert ranks[0].info()[2] == 19
    for x in ranks:
        x.close()
    # a rank without nodes: init + posts for sweeps 2, 3 + closing solve
    ranks = PeerNodeParallelDsdc.in_process(p, _cfg(2, 4), 90.0, 4)
    assert [x.info()[1:] for x in ranks] == [(1, 16), (1, 16), (0, 6), (0, 6)]
    for x in ranks:
        x.close()


def test_exchange_reset_rebases_divergence():
    import torch

    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

    p = gpu(63)
    cfg = _cfg(3, 3)
    x = PeerNodeParallelDsdc(p, cfg, 120.0, world=1, rank=0)
    a = torch.from_numpy(random_initial_state(p.grid, 2)).to(p.device)
    x.run(a, 3)
    assert x.diverged() == 0
    x.reset()
    b = torch.from_numpy(random_initial_state(p.grid, 0) * 1e140).to(p.device)
    ref = b.clone()
    x.run(b, 6)
    got = x.diverged()
    from paper_2403_20135_b200.integrators import DeviceStepper

    st = DeviceStepper(p, cfg, 120.0, serial=False)
    st.run(ref, 6)
    assert got == st.diverged() > 0
    st.close()
    x.close()


@pytest.mark.parametrize("m,k,world,parts", [(3, 3, 2, 2), (3, 3, 4, 2), (3, 3, 6, 2), (3, 2, 3, 3),
                                             (4, 4, 8, 2), (2, 3, 4, 4)])
@pytest.mark.parametrize("fused", [True, False])
def test_exchange_spectral_split_bitwise(m, k, world, parts, fused):
    """G node groups x S spectral parts over peer memory: every rank's own
    wavenumbers equal the single-GPU stepper's, bitwise."""
    import torch

    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc
    from paper_2403_20135_b200.problem import SphericalShallowWater

    ref_p = gpu(63)
    cfg = _cfg(m, k)
    u0 = torch.from_numpy(random_initial_state(ref_p.grid, 4)).to(ref_p.device)
    n_steps = 3
    ref = _stepper_result(ref_p, cfg, 120.0, u0, n_steps).reshape(3, -1)
    probs = [SphericalShallowWater(63, max_batch=4) for _ in range(world)]
    ranks = PeerNodeParallelDsdc.in_process(probs, cfg, 120.0, world, fused=fused,
                                            spectral_parts=parts)
    states = [u0.clone() for _ in ranks]
    PeerNodeParallelDsdc.run_in_stream_order(ranks, states, n_steps)
    torch.cuda.synchronize()
    covered = torch.zeros(ref.shape[1], dtype=torch.bool)
    for x, u in zip(ranks, states):
        own = torch.from_numpy(x.own_coefficients())
        got = u.reshape(3, -1)[:, own.to(u.device)]
        assert torch.equal(got, ref[:, own.to(u.device)]), (x.rank, x.part)
        covered |= own
        assert x.diverged() == 0
    assert bool(covered.all())
    for x in ranks:
        x.close()


def test_exchange_spectral_split_table_streaming():
    """T511 (TMA analysis, cp.async synthesis): 1 node group x 2 parts, all nodes batched."""
    import torch

    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc
    from paper_2403_20135_b200.problem import SphericalShallowWater

    ref_p = gpu(511, max_batch=4)
    cfg = _cfg(3, 2)
    u0 = torch.from_numpy(random_initial_state(ref_p.grid, 6)).to(ref_p.device)
    ref = _stepper_result(ref_p, cfg, 30.0, u0, 2).reshape(3, -1)
    probs = [SphericalShallowWater(511, max_batch=3) for _ in range(2)]
    ranks = PeerNodeParallelDsdc.in_process(probs, cfg, 30.0, 2, spectral_parts=2)
    states = [u0.clone() for _ in ranks]
    PeerNodeParallelDsdc.run_in_stream_order(ranks, states, 2)
    torch.cuda.synchronize()
    for x, u in zip(ranks, states):
        own = torch.from_numpy(x.own_coefficients()).to(u.device)
        assert torch.equal(u.reshape(3, -1)[:, own], ref[:, own])
        x.close()


@pytest.mark.parametrize("split", [False, True])
def test_missing_peer_post_is_an_error_not_a_hang(split):
    """a rank whose peer never posts (a killed or stalled
    process) stops waiting after the wait bound and reports which rank did not
    post, instead of spinning forever.  Rank 0 of a 2-rank exchange runs alone:
    its node kernel of sweep 2 waits for node exchange 1 (split: its ring
    kernel waits for the Fourier exchange of f_E(u0)), which rank 1 never
    posts.  One kernel waits on nothing that runs concurrently, bounded to
    250 ms.  reset() clears the error."""
    import time

    import torch

    from paper_2403_20135_b200.errors import DeviceError
    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc
    from paper_2403_20135_b200.problem import SphericalShallowWater

    cfg = _cfg(3, 3)
    if split:
        probs = [SphericalShallowWater(63, max_batch=8) for _ in range(2)]
        ranks = PeerNodeParallelDsdc.in_process(probs, cfg, 120.0, 2, spectral_parts=2)
        phases, what = range(0, 2), "Fourier exchange 1"
    else:
        p = gpu(63)
        ranks = PeerNodeParallelDsdc.in_process(p, cfg, 120.0, 2)
        phases, what = range(0, 5), "node exchange 1"
    x = ranks[0]
    x.set_wait_bound(250)
    u = torch.from_numpy(random_initial_state(x.problem.grid, 3)).to(x.problem.device)
    t0 = time.perf_counter()
    for h in phases:
        x.phase(u, h)
    with pytest.raises(DeviceError, match=f"rank 1 did not post {what}"):
        x.diverged()
    assert time.perf_counter() - t0 < 20.0
    x.reset()
    assert x.diverged() == 0
    for r in ranks:
        r.close()


def _ipc_worker(rank, world, port, split, out_path):
    import os

    import numpy as np
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc
    from paper_2403_20135_b200.problem import SphericalShallowWater

    p = SphericalShallowWater(63, device=0, max_batch=8)
    cfg = _cfg(4, 3)
    x = PeerNodeParallelDsdc(p, cfg, 120.0, spectral_parts=world if split else 1)
    x.set_wait_bound(10000)  # a protocol error fails the test instead of hanging it
    u = torch.from_numpy(random_initial_state(p.grid, 23)).to(p.device)
    x.run_serialized(u, 3)
    bad = x.diverged()  # raises DeviceError if a wait ran out
    own = x.own_coefficients()
    np.save(out_path + f".{rank}.npy", u.cpu().numpy().reshape(-1))
    np.save(out_path + f".{rank}.own.npy", own)
    assert bad == 0
    x.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("split", [False, True])
def test_two_processes_over_cuda_ipc_bitwise(tmp_path, split):
    """two processes on one GPU, each with its own plan and
    exchange, map each other's buffers through real CUDA IPC handles; the
    analysis epilogue (or the split synthesis) of one process stores into the
    other's buffer and the posts are system-scope atomics into the other's flag
    block.  The ranks take turns per half-phase (run_serialized), so every wait
    is satisfied by completed kernels of the other process.  Both ranks end
    bitwise equal to the single-GPU stepper (on their own wavenumbers when
    split)."""
    import os

    import numpy as np
    import torch
    import torch.multiprocessing as mp

    from paper_2403_20135_b200.problem import SphericalShallowWater

    world = 2
    port = 29400 + (os.getpid() % 97) + (50 if split else 0)
    out = str(tmp_path / "u")
    mp.spawn(_ipc_worker, args=(world, port, split, out), nprocs=world, join=True)
    p = SphericalShallowWater(63, device=0, max_batch=8)
    u0 = torch.from_numpy(random_initial_state(p.grid, 23)).to(p.device)
    ref = _stepper_result(p, _cfg(4, 3), 120.0, u0, 3).cpu().numpy().reshape(-1)
    p.close()
    for r in range(world):
        got = np.load(out + f".{r}.npy")
        own = np.tile(np.load(out + f".{r}.own.npy"), 3)
        assert np.array_equal(got[own], ref[own]), r


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_bench_node_parallel_path_world_one(transport):
    """The bench's multi-GPU orchestration end to end at world size 1
    (torch.distributed init, exchange construction, graphs, e2e, JSON line):
    the path `bench.py --gpus N` takes, on the one GPU this pool gives."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_PORT=str(29500 + (os.getpid() % 97) + (7 if transport == "nccl" else 0)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--node-parallel", "--transport",
                        transport, "--steps", "1", "--warmup", "1", "--no-cpu", "--no-large"],
                       capture_output=True, text=True, timeout=900, cwd=root, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["config"]["multi_gpu_transport"] == transport
    assert line["config"]["finite"] and line["value"] > 0 and line["e2e"]["value"] > 0
