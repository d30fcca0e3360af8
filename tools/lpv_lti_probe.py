import sys, numpy as np, scipy.signal as sig, time
sys.path.insert(0, '/root/repo')
from paper_2604_12505_b200.lpv import identify, normalise
def _rng(s): return np.random.Generator(np.random.Philox(s))
r = _rng(40)
A = r.normal(0, 1, (4, 4)); A = 0.9 * A / np.abs(np.linalg.eigvals(A)).max()
B, Cm = r.normal(0, 1, (4, 3)), r.normal(0, 1, (3, 4))
K = 300; us = [r.normal(size=(K, 3))]
_, y, _ = sig.dlsim((A, B, Cm, np.zeros((3, 3)), 0.05), us[0])
un, yn, _ = normalise(us, [y])
for kw in [dict(lbfgs_iters=400, lti_iters=800), dict(lbfgs_iters=2000, lti_iters=1500), dict(lbfgs_iters=2000, lti_iters=1500, ftol=0.0)]:
    t0=time.time(); res = identify(un, yn, restarts=2, adam_iters=300, seed=6, lr=3e-3, **kw)
    print(kw, res["bfr_lti"], res["bfr"], "%.1fs"%(time.time()-t0), flush=True)
