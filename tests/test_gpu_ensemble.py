"""Multi-rank ensemble with REAL SPH rollouts: two processes on one GPU, each
running its shard of the global rollout ids through the C ABI, one gather of the dataset
(y, u_applied, status) over torch.distributed (gloo here: one GPU cannot host an NCCL
communicator of two ranks).  The gathered dataset must be bitwise equal to the single-process
batch of all rollouts: each rollout's inputs and arithmetic depend only on its global id."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import sph_inputs as si

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tank():
    t = si.make_tank(1.0)
    import oracle as O
    s = O.settle(t, seconds=0.5)
    return t, np.concatenate([s.pos, s.vel], 1).astype(np.float32)


def _worker(rank, world, port, n_total, K, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_12505_b200.ensemble import run_ensemble
    t, pv = _tank()
    y, ua, st = run_ensemble(t.params, pv, t.ghost_b, n_total, K, kind, rank=rank, world=world,
                             device=0, rebin_every=0, skin=0.15 * t.params.h)
    if rank == 0:
        q.put((y.cpu().numpy(), ua.cpu().numpy(), st.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n_total", [("excitation", 6), ("profiles", 5)])
def test_two_rank_ensemble_equals_single_process(kind, n_total):
    from paper_2604_12505_b200.ensemble import run_ensemble
    K, world = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, K, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    y2, ua2, st2 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    t, pv = _tank()
    y1, ua1, st1 = run_ensemble(t.params, pv, t.ghost_b, n_total, K, kind, rebin_every=0,
                                skin=0.15 * t.params.h)
    assert np.array_equal(y2, y1.cpu().numpy())
    assert np.array_equal(ua2, ua1.cpu().numpy())
    assert np.array_equal(st2, st1.cpu().numpy()) and st2.max() == 0
    if kind == "profiles":   # PD law active: torque = Kp (theta_ref - theta) - Kd thetadot
        assert np.abs(ua2[..., 2]).max() > 0
