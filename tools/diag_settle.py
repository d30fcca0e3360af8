#!/usr/bin/env python3
import math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si
import oracle as O
from paper_2604_12505_b200 import SphContext
for ell, secs in ((1.0, 2.0), (4.0, 0.5)):
    t = si.make_tank(ell, jitter=0.02, seed=11).snapped(); sp = t.params
    n = int(round(secs / sp.dt))
    for path in (0, 1):
        for skin in (0.1, 0.3):
            ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=skin * sp.h, rebuild_path=path)
            ctx.settle(math.exp(-10 * sp.dt), n)
            pv, rho = ctx.get_particles(0, with_rho=True)
            steps, reb = ctx.counters(); ctx.close()
            print(f"GPU ell {ell} path {path} skin {skin}: max|v| {np.abs(pv[:,2:]).max():.3e}  rho {rho.min()/sp.rho0:.5f}..{rho.max()/sp.rho0:.5f}  rebuilds {reb[0]}/{steps[0]}")
    if ell == 1.0:
        ref = O.State.from_tank(t); rr = ref.step(n=n, damping=math.exp(-10 * sp.dt), pin_body=True, want_rho=True)
        print(f"ORC ell {ell}: max|v| {np.abs(ref.vel).max():.3e}  rho {rr.min()/sp.rho0:.5f}..{rr.max()/sp.rho0:.5f}")
