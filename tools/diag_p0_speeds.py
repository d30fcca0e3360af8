#!/usr/bin/env python3
"""P0 profile-1 closed loop: relative fluid speed statistics, GPU vs oracle (long horizon:
chaotic, so statistics, not trajectories, are compared)."""
import os, sys, math, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle as O
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
t = si.make_tank(1.0, n_first=666); sp = t.params
s = O.settle(t, seconds=2.0)
pv0 = np.concatenate([s.pos, s.vel], 1).astype(np.float32)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
u, th = si.profile(1, K)
ctx = SphContext(sp, pv0, t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.15 * sp.h)
ref = O.State(sp, pv0[:, :2].astype(np.float64), pv0[:, 2:].astype(np.float64), t.ghost_b)
def stats(vel, body):
    rel = vel - body[3:5]
    v = np.sqrt((rel ** 2).sum(1))
    return v.max(), np.percentile(v, 99), np.median(v)
for k0 in range(0, K, 20):
    uu = u[k0:k0 + 20].astype(np.float32)
    tt = th[k0:k0 + 20].astype(np.float32)
    ctx.rollout(uu[None], theta_ref=tt[None], Kp=sp.Kp, Kd=sp.Kd)
    ref.rollout(uu.astype(np.float64), sp.n_sub, theta_ref=tt.astype(np.float64), Kp=sp.Kp, Kd=sp.Kd)
    g = stats(ctx.get_particles(0)[:, 2:].astype(np.float64), ctx.get_body_state()[0])
    o = stats(ref.vel, ref.body)
    print(f"t={(k0 + 20) * 0.05:5.1f}s  GPU max/p99/med {g[0]:.4f} {g[1]:.4f} {g[2]:.4f}   oracle {o[0]:.4f} {o[1]:.4f} {o[2]:.4f}")
