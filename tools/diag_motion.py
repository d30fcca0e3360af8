#!/usr/bin/env python3
"""Diagnostic: settle a C2 tank, then run a small C3-like batch; print motion statistics."""
import math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
t = si.make_tank(4.0); sp = t.params
one = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1)
one.settle(math.exp(-10 * sp.dt), int(2.0 / sp.dt))
pv, rho = one.get_particles(0, with_rho=True)
print("settled: max|v| %.3e  rho/rho0 min %.5f max %.5f" % (np.abs(pv[:, 2:]).max(), rho.min() / sp.rho0, rho.max() / sp.rho0))
one.close()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=0.1 * sp.h)
u = si.ensemble_inputs(range(B), 8)[0]
y, _ = ctx.rollout(u)
steps, reb = ctx.counters()
vs = [np.abs(ctx.get_particles(b)[:, 2:]).max() for b in range(min(B, 8))]
print("B %d substeps/rebuild %.1f  max|v| first rollouts %s  y checksum %.9e" % (B, steps.mean() / reb.mean(), np.round(vs, 5), np.abs(y).sum()))
