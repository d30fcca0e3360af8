"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: sharding by global rollout id,
inputs independent of the world size, and the trajectory gather in global-id order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import sph_inputs as si
from paper_2604_12505_b200.ensemble import gather_trajectories, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_ids_once():
    for n, w in ((8192, 8), (10, 3), (1, 2), (0, 4)):
        ids = [g for r in range(w) for g in shard(n, w, r)]
        assert ids == list(range(n))


def test_inputs_depend_only_on_global_id():
    a = si.ensemble_inputs(range(0, 6), 20)[0]
    b = np.concatenate([si.ensemble_inputs(shard(6, 2, r), 20)[0] for r in range(2)])
    assert np.array_equal(a, b)
    u1, t1 = si.profile_inputs([5, 4099], 8192, 50)
    u2, t2 = si.profile_inputs([4099], 8192, 50)
    assert np.array_equal(u1[1], u2[0]) and np.array_equal(t1[1], t2[0])


def _worker(rank, world, port, n_total, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = list(shard(n_total, world, rank))
    # stand-in for each rollout's trajectory: a deterministic function of its global id only
    u = torch.from_numpy(si.ensemble_inputs(ids, K)[0]) if ids else torch.zeros((0, K, 3))
    y = torch.cat([u, 2 * u], dim=2)
    out = gather_trajectories(y)
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [6, 7])
def test_gloo_gather_matches_single_rank(n_total):
    K, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    u = si.ensemble_inputs(range(n_total), K)[0]
    assert np.array_equal(got, np.concatenate([u, 2 * u], axis=2))
