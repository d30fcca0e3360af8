"""C4 tank (ell = 42), lattice start, N substeps through sph_step (per-substep launches) with the
bench's skin policy -- for ncu launch lists of the large-tank substep."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si
from paper_2604_12505_b200 import SphContext
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t = si.make_tank(42.0)
sp = t.params
ctx = SphContext(sp, t.pv32(), t.ghost_b, n_rollouts=1, rebin_every=0, skin=0.15 * sp.h,
                 skin_max=0.8 * sp.h, skin_mode=1)
ctx.step(np.array([[5.0, 0.0, 0.0]], np.float32), n)
print("ok", ctx.counters(), flush=True)
