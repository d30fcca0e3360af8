"""Bitwise A/B of two library builds on the resident path: python tools/ab_bits.py OUT.npz runs
C1 (B = 3) and C2 (B = 2) rollouts through the library SPH_LIB_PATH points at and saves the
results; python tools/ab_bits.py --cmp A.npz B.npz compares two such files bit for bit."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise equal" if not bad else f"DIFFER: {bad}")
    sys.exit(1 if bad else 0)

import sph_inputs as si  # noqa: E402
from paper_2604_12505_b200 import SphContext  # noqa: E402

out = {}
for ell, B, pvf in ((1.0, 3, None), (4.0, 2, "bench_data/settled_ell4.npz")):
    t = si.make_tank(ell)
    pv = t.pv32() if pvf is None else np.ascontiguousarray(np.load(pvf)["pv"], dtype=np.float32)
    ctx = SphContext(t.params, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=0.15 * t.params.h,
                     exec_path=3, skin_max=0.5 * t.params.h)
    u = si.ensemble_inputs(range(B), 3)[0] * (10.0 if ell == 1.0 else 1.0)
    y, _ = ctx.rollout(u)
    ctx.step(u[:, 0], 37)
    tag = f"l{ell:g}"
    out[tag + "_y"] = y
    out[tag + "_body"] = ctx.get_body_state()
    out[tag + "_pv"] = np.stack([ctx.get_particles(b) for b in range(B)])
    out[tag + "_reb"] = ctx.counters()[1]
    print(tag, "path", ctx.exec_path(), "rebuilds", ctx.counters()[1])
    ctx.close()
# small path (per-rollout rebuild branch, k_nlist_density) on 4 C2 tanks, 3 ticks
t = si.make_tank(4.0)
pv = np.ascontiguousarray(np.load("bench_data/settled_ell4.npz")["pv"], dtype=np.float32)
ctx = SphContext(t.params, pv, t.ghost_b, n_rollouts=4, rebin_every=0, skin=0.15 * t.params.h,
                 exec_path=1, rebuild_path=1, skin_max=0.5 * t.params.h)
y, _ = ctx.rollout(si.ensemble_inputs(range(4), 3)[0] * 20.0)
out["small_y"] = y
out["small_pv"] = np.stack([ctx.get_particles(b, with_rho=True)[1] for b in range(4)])
out["small_reb"] = ctx.counters()[1]
print("small path rebuilds", ctx.counters()[1])
ctx.close()
# large tank (bsplit > 1: fused body kernel), per-particle half-skins as the C4 bench
t = si.make_tank(42.0)
ctx = SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.15 * t.params.h,
                 skin_max=0.8 * t.params.h, skin_mode=1)
ctx.step(np.array([[5.0, 2.0, 1.0]], np.float32), 60)
out["l42_body"] = ctx.get_body_state()
out["l42_pv"] = ctx.get_particles(0)
out["l42_reb"] = ctx.counters()[1]
y, _ = ctx.rollout(np.array([[[3.0, -1.0, 0.5]]], np.float32))   # one captured tick (2100 substeps)
out["l42_y"] = y
out["l42_body2"] = ctx.get_body_state()
out["l42_pv2"] = ctx.get_particles(0)
out["l42_reb2"] = ctx.counters()[1]
print("l42 path", ctx.exec_path(), "rebuilds", ctx.counters()[1], "launches/tick", ctx.launches_per_tick())
ctx.close()
np.savez(sys.argv[1], **out)
