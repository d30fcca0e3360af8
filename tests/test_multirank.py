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


def _ds_worker(rank, world, port, n_total, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_12505_b200.ensemble import gather_dataset
    ids = list(shard(n_total, world, rank))
    u = torch.from_numpy(si.ensemble_inputs(ids, K)[0]) if ids else torch.zeros((0, K, 3))
    y = torch.cat([u, -u], dim=2)                      # stand-in y [B, K, 6], u_applied = u
    st = torch.tensor([g % 3 for g in ids], dtype=torch.int32)
    yg, ug, sg = gather_dataset(y, u, st)
    if rank == 0:
        q.put((yg.numpy(), ug.numpy(), sg.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_gather_dataset_y_u_status():
    """The dataset gather of the C5 path (y, u_applied and the per-rollout status in one
    collective) returns every rank's rows in global-id order."""
    n_total, K, world = 7, 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ds_worker, args=(r, world, port, n_total, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    yg, ug, sg = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    u = si.ensemble_inputs(range(n_total), K)[0]
    assert np.array_equal(yg, np.concatenate([u, -u], axis=2)) and np.array_equal(ug, u)
    assert sg.tolist() == [g % 3 for g in range(n_total)]


# ---- domain decomposition: slab ranges and the in-place padded all-gather ----

def test_slab_ranges():
    from paper_2604_12505_b200.parallel import slab_ranges, n_partials, DD_ALIGN
    for n, w in ((9261, 2), (9261, 3), (1_000_000, 8), (4096, 4)):
        chunk, rng = slab_ranges(n, w)
        assert chunk % DD_ALIGN == 0 and rng[0][0] == 0 and rng[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))
        assert w * chunk >= n and w * chunk // 32 >= n_partials(n)


def _dd_worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_12505_b200.parallel import slab_ranges, all_gather_inplace
    chunk, rng = slab_ranges(n, world)
    lo, hi = rng[rank]
    # each rank fills only its own slab of a padded buffer, as sph_dd_phase does
    aux = torch.zeros((world * chunk, 2))
    aux[lo:hi] = torch.arange(lo, hi, dtype=torch.float32)[:, None] * torch.tensor([1.0, -1.0])
    part = torch.zeros((world * chunk // 32, 4), dtype=torch.float64)
    part[lo // 32:(hi + 31) // 32] = float(rank + 1)
    all_gather_inplace(dist, aux, rank)
    all_gather_inplace(dist, part, rank)
    q.put((rank, aux[:n].numpy().copy(), part.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [9261, 5000])
def test_gloo_dd_exchange(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dd_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2604_12505_b200.parallel import slab_ranges
    chunk, rng = slab_ranges(n, world)
    ref = np.arange(n, dtype=np.float32)[:, None] * np.array([1.0, -1.0], np.float32)
    for rank, aux, part in out:
        assert np.array_equal(aux, ref)                       # every rank holds the whole array
        for r, (lo, hi) in enumerate(rng):
            assert np.all(part[lo // 32:(hi + 31) // 32] == r + 1)
