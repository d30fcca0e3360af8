#!/usr/bin/env python3
"""Identification probes (GPU): known-LPV data with several optimiser budgets, and the SPH
dataset of the bench's LPV workload.  Prints BFRs and wall times."""
import os, sys, time, math
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import lpv as OL
from paper_2604_12505_b200.lpv import identify, normalise

def rng(s): return np.random.Generator(np.random.Philox(s))
def theta(seed, a1=0.1):
    r = rng(seed)
    P = {n: r.normal(0, 0.4, s) for n, s in OL.SIZES}
    A = r.normal(0, 1, (4, 4)); P["A0"] = 0.85 * A / np.abs(np.linalg.eigvals(A)).max()
    P["A1"] = r.normal(0, a1, (4, 4))
    P["B1"] = r.normal(0, a1, (4, 3)); P["C1"] = r.normal(0, a1, (3, 4))
    return OL.pack(P)
th = theta(30, a1=float(os.environ.get('A1', '0.1'))); r = rng(31); K = 300
us = [r.normal(size=(K, 3)) for _ in range(2)]
ys = [OL.simulate(th, np.zeros(4), u)[0] for u in us]
un, yn, _ = normalise(us, ys)
for cfg in [dict(restarts=4, adam_iters=600, lbfgs_iters=400, lti_iters=300, lr=3e-3),
            dict(restarts=8, adam_iters=2000, lbfgs_iters=1500, lti_iters=1000, lr=3e-3),
            ]:
    t0 = time.time()
    res = identify(un, yn, seed=5, **cfg)
    print(cfg, "bfr_lti %.2f bfr %.2f" % (res["bfr_lti"], res["bfr"]), np.round(res["bfr_all"], 1), "%.1fs" % (time.time() - t0), flush=True)
