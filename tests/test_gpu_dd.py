"""Spatial domain decomposition of one tank (sph_set_domain / sph_dd_phase,
paper_2604_12505_b200.parallel) on one GPU: W slabs in one process (parallel.LocalGroup; the
multi-process NCCL exchange is covered on CPU by tests/test_multirank.py) advance the tank
bitwise identically to the undecomposed context, and the decomposed state matches the oracle
after one step."""
import numpy as np
import pytest

import oracle as O
import sph_inputs as si

pytestmark = pytest.mark.gpu
BODY = [0.01, -0.02, 0.3, 0.02, -0.01, 0.05]


def _ctx(t, **kw):
    """Single-rollout context on the per-substep kernel path (exec_path 1): the decomposition
    reuses those kernels, so the undecomposed reference must run them too (auto would pick the
    resident clusters for one rollout, whose float32 summation order differs)."""
    from paper_2604_12505_b200 import SphContext
    kw.setdefault("exec_path", 1)
    c = SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=1, **kw)
    c.set_body_state(np.array([t.body]))
    return c


@pytest.mark.parametrize("W,adaptive", [(2, False), (3, True), (1, True)])
def test_decomposed_bitwise_equals_single(W, adaptive):
    from paper_2604_12505_b200.parallel import LocalGroup
    t = si.moving_tank(4.0, seed=7, vel=0.02, body=BODY)          # C2: 9,261 particles
    kw = dict(rebin_every=0, skin=0.3 * t.params.h) if adaptive else dict(rebin_every=1)
    ref = _ctx(t, **kw)
    grp = LocalGroup([_ctx(t, **kw) for _ in range(W)])
    r = np.random.Generator(np.random.Philox(3))
    for k in range(25):
        u = (r.normal(size=3) * 20.0).astype(np.float32)
        ref.step(u[None], 1)
        grp.substep(u)
    pv_ref = ref.get_particles(0)
    body_ref = ref.get_body_state()[0]
    for p in grp.parts:
        assert np.array_equal(p.ctx.get_particles(0), pv_ref)
        assert np.array_equal(p.ctx.get_body_state()[0], body_ref)
        assert p.ctx.get_status()[0][0] == 0
    if adaptive:
        assert grp.parts[0].ctx.counters()[1][0] == ref.counters()[1][0]


def test_decomposed_one_step_matches_oracle():
    from paper_2604_12505_b200.parallel import LocalGroup
    t = si.moving_tank(4.0, seed=8, vel=0.02, body=BODY)
    grp = LocalGroup([_ctx(t) for _ in range(2)])
    u = (5.0, 2.0, 1.0)
    grp.substep(np.array(u, np.float32))
    ref = O.State.from_tank(t)
    ref.step(u)
    pv = grp.parts[1].ctx.get_particles(0).astype(np.float64)
    scale = np.abs(ref.pos).max()
    assert np.abs(pv[:, :2] - ref.pos).max() <= 1e-5 * scale
    bg = grp.parts[0].ctx.get_body_state()[0]
    assert np.abs(bg[:3] - ref.body[:3]).max() <= 1e-5 * max(np.abs(ref.body[:3]).max(), 1.0)


def test_domain_validation():
    from paper_2604_12505_b200 import SphError
    from paper_2604_12505_b200.parallel import slab_ranges
    t = si.make_tank(4.0)
    c = _ctx(t)
    L = c.L
    assert L.sph_set_domain(c.ctx, 100, 2048) != 0          # unaligned start
    assert L.sph_set_domain(c.ctx, 0, c.N + 1) != 0         # beyond N
    assert L.sph_set_domain(c.ctx, 1024, 1024) != 0         # empty
    assert L.sph_set_domain(c.ctx, 1024, c.N) == 0
    with pytest.raises(ValueError):
        slab_ranges(569, 2)                                  # C1 is one slab's worth
    c.close()
    t2 = si.make_tank(1.0)
    from paper_2604_12505_b200 import SphContext
    c2 = SphContext(t2.params, t2.pv32(), t2.ghost_b, n_rollouts=2)
    assert c2.L.sph_set_domain(c2.ctx, 0, c2.N) != 0         # more than one rollout
    c2.close()


def _dd_rank(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_12505_b200.parallel import DistributedTank
    t = si.moving_tank(4.0, seed=7, vel=0.02, body=BODY)
    ctx = _ctx(t, rebin_every=0, skin=0.3 * t.params.h)
    tank = DistributedTank(ctx)
    r = np.random.Generator(np.random.Philox(5))
    for k in range(12):
        tank.substep((r.normal(size=3) * 20.0).astype(np.float32))
    torch.cuda.synchronize()
    q.put((rank, ctx.get_particles(0), ctx.get_body_state()[0]))
    ctx.close()
    dist.destroy_process_group()


def test_distributed_tank_two_processes():
    """DistributedTank across two processes (gloo, host-staged all-gathers; both processes on
    this one device, nothing on the device waits for the other process): both end with the
    single-context trajectory, bitwise."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    procs = [ctxm.Process(target=_dd_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    t = si.moving_tank(4.0, seed=7, vel=0.02, body=BODY)
    ref = _ctx(t, rebin_every=0, skin=0.3 * t.params.h)
    r = np.random.Generator(np.random.Philox(5))
    for k in range(12):
        ref.step((r.normal(size=3) * 20.0).astype(np.float32)[None], 1)
    pv, body = ref.get_particles(0), ref.get_body_state()[0]
    for rank, pvr, br in out:
        assert np.array_equal(pvr, pv) and np.array_equal(br, body)
