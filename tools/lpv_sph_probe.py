#!/usr/bin/env python3
"""LPV identification on the bench's SPH dataset with reduced budgets (tuning probe)."""
import os, sys, time, math
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
from paper_2604_12505_b200 import lpv as LP
t = si.make_tank(1.0, n_first=666); sp = t.params
ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.5 * sp.h)
ctx.settle(math.exp(-10.0 * sp.dt), int(2.0 / sp.dt))
pv0 = ctx.get_particles(0)
u = si.excitation(3000, K=2200).astype(np.float32)[None]
y, _ = ctx.rollout(u)
us = [u[0].astype(np.float64)]; ys = [np.asarray(y)[0, :, 3:6].astype(np.float64)]
print("y rms", np.sqrt((ys[0]**2).mean(0)), "y end", ys[0][-1], "u rms", np.sqrt((us[0]**2).mean(0)))
for center in (False,):
    un, yn, sc = LP.normalise(us, ys, center=center)
    th = LP.arx_init(un, yn)
    prob = LP.LpvProblem(1, un, yn); P = np.zeros((1, LP.NT + 4)); P[0, :LP.NT] = th; P[0, LP.NT:LP.NT+3] = yn[0][0]
    prob.set_params(P); yh = prob.simulate()[0, 0].cpu().numpy()
    print("center", center, "ARX init BFR", LP.bfr(yn[0], yh))
    for cfg in [dict(restarts=8, adam_iters=500, lbfgs_iters=500, lti_iters=500, lr=1e-3),
                dict(restarts=8, adam_iters=2000, lbfgs_iters=2000, lti_iters=2000, lr=1e-3)]:
        t0 = time.time()
        res = LP.identify(un, yn, seed=0, **cfg)
        print(cfg, "bfr_lti %.2f bfr %.2f" % (res["bfr_lti"], res["bfr"]), np.round(res["bfr_all"], 1), "evals", res["n_evals"], "%.1fs" % (time.time() - t0), flush=True)
