"""Parity of the benchmark's own C3 path (SURVEY 8(c) tolerances, 8(d) C3 recipe).

bench.py's default line runs 1024 rollouts of the C2 tank (l = 4: 9,261 fluid + 944 ghosts) from
the oracle-settled snapshot bench_data/settled_ell4.npz, open-loop excitation inputs,
adaptive Verlet lists with skin 0.15 h, one CUDA launch sequence per slow tick of 200 substeps.
Here that exact configuration (batch size, skin, start state, inputs, launch path) runs three
ticks (600 substeps, mixed rebuild / no-rebuild substeps); rollouts 0, B/2 and B-1 are compared
with the float64 oracle run from the same float32 start on the same inputs:
  * body trajectory y_k (Eq. dataset) per channel <= 1e-3 (north star),
  * final particle positions <= 1e-5 relative to max |x| (north star's one-step bar, kept here
    over 600 substeps from a settled start),
and each of those rollouts must be bitwise equal to the same rollout run alone (B = 1) through
the same execution path (dataset D_N independent of the batch)."""
import os

import numpy as np
import pytest

import oracle as O
import sph_inputs as si

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rel(a, b, floor=0.0):
    return np.abs(a - b).max() / max(np.abs(b).max(), floor)


@pytest.fixture(scope="module")
def c3_start():
    t = si.make_tank(4.0)
    d = np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))
    pv = np.ascontiguousarray(d["pv"], dtype=np.float32)
    assert pv.shape == (t.n_fluid, 4)
    return t, pv


@pytest.mark.parametrize("exec_path", [1, 3])
def test_c3_bench_path_three_ticks_vs_oracle_and_batch_invariance(c3_start, exec_path):
    from paper_2604_12505_b200 import SphContext
    t, pv = c3_start
    sp = t.params
    B, K = 1024, 3
    ids = [0, B // 2, B - 1]
    u = si.ensemble_inputs(range(B), K)[0]
    kw = dict(rebin_every=0, skin=0.15 * sp.h, exec_path=exec_path)
    ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, **kw)
    y, ua = ctx.rollout(u)
    body = ctx.get_body_state()
    st = ctx.get_status()[0]
    steps, reb = ctx.counters()
    parts = {b: ctx.get_particles(b) for b in ids}
    ctx.close()
    assert st.max() == 0
    assert np.all(steps == K * sp.n_sub)
    # the adaptive lists really were rebuilt inside the window (mixed substeps)
    assert reb.min() >= 1 and reb.max() < K * sp.n_sub
    for b in ids:
        ref = O.State(sp, pv[:, :2].astype(np.float64), pv[:, 2:].astype(np.float64), t.ghost_b)
        yo, uo = ref.rollout(u[b].astype(np.float64), sp.n_sub)
        yf = np.concatenate([y[b], body[b][None].astype(np.float32)], 0).astype(np.float64)
        yr = np.concatenate([yo, ref.body[None]], 0)
        for c in range(6):
            assert _rel(yf[:, c], yr[:, c], 1e-12) <= 1e-3, (b, c, _rel(yf[:, c], yr[:, c], 1e-12))
        assert _rel(parts[b][:, :2], ref.pos) <= 1e-5, (b, _rel(parts[b][:, :2], ref.pos))
        assert np.array_equal(ua[b], u[b])
        one = SphContext(sp, pv, t.ghost_b, n_rollouts=1, **kw)
        y1, _ = one.rollout(u[b:b + 1])
        assert np.array_equal(y1[0], y[b]), b
        assert np.array_equal(one.get_particles(0), parts[b]), b
        assert np.array_equal(one.get_body_state()[0], body[b]), b
        one.close()


def test_c5_path_profiles_pd_vs_oracle_and_batch_invariance(c3_start):
    """The C5 configuration's path (manoeuvre profiles 1 and 2 under the PD law,
    P:364-386) on the small-rollout graph path (B = 512 >= the per-rollout rebuild threshold):
    3 ticks from the settled C2 snapshot; rollout 0 (profile 1) and rollout B-1 (profile 2) against
    the float64 oracle on the same inputs (body trajectory and the applied PD torque <= 1e-3), and
    bitwise equal to the same rollout alone (B = 1, multi-kernel path)."""
    from paper_2604_12505_b200 import SphContext
    t, pv = c3_start
    sp = t.params
    B, K = 512, 3
    # a window where both profiles act: from the tick before rollout B-1's first pulse (profile
    # 2 starts at 2 +- 1 s); profile 1 thrusts from t = 0 (inputs taken mid-profile from rest)
    u_all, th_all = si.profile_inputs(range(B), B, 80)
    k0 = max(0, int(np.argmax(np.abs(u_all[B - 1]).sum(1) > 0)) - 1)
    u = np.ascontiguousarray(u_all[:, k0:k0 + K])
    th = np.ascontiguousarray(th_all[:, k0:k0 + K])
    kw = dict(rebin_every=0, skin=0.15 * sp.h, skin_max=0.5 * sp.h, exec_path=1)
    ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, **kw)
    y, ua = ctx.rollout(u, theta_ref=th, Kp=sp.Kp, Kd=sp.Kd)
    body = ctx.get_body_state()
    assert ctx.get_status()[0].max() == 0
    ctx.close()
    for b in (0, B - 1):
        ref = O.State(sp, pv[:, :2].astype(np.float64), pv[:, 2:].astype(np.float64), t.ghost_b)
        yo, uo = ref.rollout(u[b].astype(np.float64), sp.n_sub, theta_ref=th[b].astype(np.float64),
                             Kp=sp.Kp, Kd=sp.Kd)
        yf = np.concatenate([y[b], body[b][None].astype(np.float32)], 0).astype(np.float64)
        yr = np.concatenate([yo, ref.body[None]], 0)
        # errors relative to the trajectory's own scale: the larger of |r| and R |theta| for the
        # pose, of |rdot| and R |thetadot| for the rates (angles divided by R).  Under a profile the thrust acts through
        # the CoM along one axis, so the other components are symmetry-zero up to float32 noise
        # (~1e-11 m, ~1e-9 rad), which a per-component relative error would amplify
        rs = max(np.abs(yr[:, 0:2]).max(), sp.R * np.abs(yr[:, 2]).max())   # displacement scale
        vs = max(np.abs(yr[:, 3:5]).max(), sp.R * np.abs(yr[:, 5]).max())   # speed scale
        assert rs > 1e-6 and vs > 1e-5, (rs, vs)   # the manoeuvre has started
        scale = [rs, rs, rs / sp.R, vs, vs, vs / sp.R]
        for c in range(6):
            assert _rel(yf[:, c], yr[:, c], scale[c]) <= 1e-3, (b, c, _rel(yf[:, c], yr[:, c], scale[c]))
        assert _rel(ua[b], uo, 1e-12) <= 1e-3, b
        one = SphContext(sp, pv, t.ghost_b, n_rollouts=1, **kw)
        y1, ua1 = one.rollout(u[b:b + 1], theta_ref=th[b:b + 1], Kp=sp.Kp, Kd=sp.Kd)
        assert np.array_equal(y1[0], y[b]) and np.array_equal(ua1[0], ua[b]), b
        one.close()
