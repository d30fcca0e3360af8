#!/usr/bin/env python3
"""LTI-stage tuning on the SPH dataset: ARX init -> Adam(lr, N) -> L-BFGS(M); BFR per channel."""
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
u = si.excitation(3000, K=2200).astype(np.float32)[None]
y, _ = ctx.rollout(u)
us = [u[0].astype(np.float64)]; ys = [np.asarray(y)[0, :, 3:6].astype(np.float64)]
np.savez(os.path.join(ROOT, "gpurun_out", "lpv_data.npz"), u=us[0], y=ys[0])
un, yn, sc = LP.normalise(us, ys)
th = LP.arx_init(un, yn)
print("ARX A", np.round(LP.block(th, "A0"), 4).tolist(), "B", np.round(LP.block(th, "B0"), 5).tolist())
for lr, N, M in [(1e-3, 2000, 500), (1e-2, 2000, 500), (3e-3, 2000, 2000), (1e-2, 4000, 2000)]:
    R = 4
    prob = LP.LpvProblem(R, un, yn)
    P = np.zeros((R, LP.NT + 4)); P[:, :LP.NT] = th; P[:, LP.NT:LP.NT+3] = yn[0][0]
    rng = np.random.Generator(np.random.Philox(1))
    P[1:, LP.NT - 57 - 40 + 0: LP.NT - 57 - 40 + 40] = 0   # M1 stays 0
    P[1:, 3 * 4 + 3] = [0.5, 0.0, -0.5]                    # slosh pole variants
    prob.set_params(P)
    tr = np.zeros(prob.n, bool); tr[:40] = True; tr[LP.NT:] = True
    prob.set_mask(tr)
    t0 = time.time(); prob.adam(N, lr=lr); ne = prob.lbfgs(M)
    yh = prob.simulate().cpu().numpy()
    print(f"lr {lr} adam {N} lbfgs {M}: evals {ne}", [np.round(LP.bfr(yn[0], yh[r, 0]), 1).tolist() for r in range(R)], "%.1fs" % (time.time() - t0), flush=True)
