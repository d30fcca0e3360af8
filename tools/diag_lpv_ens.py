"""Status of the 8-rollout P0 identification ensemble (110 s excitation) on two execution paths."""
import math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
t = si.make_tank(1.0, n_first=666)
sp = t.params
ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.5 * sp.h)
ctx.settle(math.exp(-10.0 * sp.dt), int(2.0 / sp.dt))
pv0 = ctx.get_particles(0)
ctx.close()
u = si.ensemble_inputs(range(8), 2200)[0]
for ex in (3, 2, 1):
    c = SphContext(sp, pv0, t.ghost_b, n_rollouts=8, rebin_every=0, skin=0.5 * sp.h, exec_path=ex)
    y, _ = c.rollout(u)
    st, bs, bp = c.get_status()
    print(ex, c.exec_path(), st.tolist(), bs.tolist(), bp.tolist(), flush=True)
    c.close()
