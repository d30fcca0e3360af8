#!/usr/bin/env python3
"""Rebuild rate vs relative fluid speed along the profile-1 closed loop of the C2 tank."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
t = si.make_tank(4.0); sp = t.params
pv0 = np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"].astype(np.float32)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
u, th = si.profile(1, K)
ctx = SphContext(sp, pv0, t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.15 * sp.h)
prev = 0
thr = 0.45 * 0.15 * sp.h
for k in range(K):
    ctx.rollout(u[None, k:k + 1].astype(np.float32), theta_ref=th[None, k:k + 1].astype(np.float32), Kp=sp.Kp, Kd=sp.Kd)
    if k % 20 == 19:
        steps, reb = ctx.counters()
        pv = ctx.get_particles(0)
        body = ctx.get_body_state()[0]
        rel = pv[:, 2:] - body[3:5]
        sp_rel = np.sqrt((rel ** 2).sum(1))
        print(f"t={k * 0.05 + 0.05:5.2f}s rebuilds/tick {(int(reb[0]) - prev) / 20:6.1f}  max|v-rd| {sp_rel.max():.4f} m/s "
              f"p99 {np.percentile(sp_rel, 99):.4f}  -> expected substeps/rebuild {thr / (sp_rel.max() * sp.dt):7.1f}  |rd| {np.hypot(*body[3:5]):.4f} thd {body[5]:.4f}")
        prev = int(reb[0])
