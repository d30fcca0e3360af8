#!/usr/bin/env python3
"""Speed distribution of the C4 tank (ell = 42) after a damped settle and after excitation
ticks: which particles trip the Verlet bound (rebuild every ~2 substeps at skin 0.15h)."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si  # noqa: E402
from paper_2604_12505_b200 import SphContext  # noqa: E402

settle_s = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
t = si.make_tank(42.0)
sp = t.params


def report(tag, pv):
    sp_ = np.hypot(pv[:, 2], pv[:, 3])
    r = np.hypot(pv[:, 0], pv[:, 1])
    top = np.argsort(sp_)[-6:][::-1]
    print(f"{tag}: max {sp_.max():.3e} p99.9 {np.quantile(sp_, 0.999):.3e} p99 {np.quantile(sp_, 0.99):.3e} "
          f"median {np.median(sp_):.3e} n>0.1 {(sp_ > 0.1).sum()} n>0.03 {(sp_ > 0.03).sum()}")
    for i in top:
        print(f"   id {i}: |v| {sp_[i]:.3e} x {pv[i, 0]:+.4f} y {pv[i, 1]:+.4f} r {r[i]:.4f} (R - r)/s "
              f"{(0.2 - r[i]) / sp.spacing:.2f}")


ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.15 * sp.h)
report("lattice", ctx.get_particles(0))
n = int(round(settle_s / sp.dt))
ctx.settle(math.exp(-10.0 * sp.dt), n)
report(f"settled {settle_s} s", ctx.get_particles(0))
steps0, reb0 = ctx.counters()
ctx.step(np.zeros((1, 3), np.float32), 200)
steps1, reb1 = ctx.counters()
report("200 free substeps", ctx.get_particles(0))
print("substeps per rebuild (free):", (steps1 - steps0) / max(reb1 - reb0, 1))
u = si.ensemble_inputs([0], 2)[0]
ctx.rollout(u)
steps2, reb2 = ctx.counters()
report("2 excitation ticks", ctx.get_particles(0))
print("substeps per rebuild (excited):", (steps2 - steps1) / max(reb2 - reb1, 1))
ctx.close()
