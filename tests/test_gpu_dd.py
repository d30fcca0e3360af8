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
    from paper_2604_12505_b200 import SphContext
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
