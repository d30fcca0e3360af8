"""C3 batch (1024 rollouts, settled C2 start) with a rebuild every substep (rebin_every = 1):
every substep runs k_rebuild_small + k_nlist_density for all rollouts -- for ncu captures of the
list-build kernel (e.g. -k regex:k_nlist_density -s 2 -c 1)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si
from paper_2604_12505_b200 import SphContext

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B = 1024
t = si.make_tank(4.0)
sp = t.params
pv = np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32)
ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=1, skin=0.5 * sp.h)
u = np.tile(np.array([[5.0, 2.0, 1.0]], np.float32), (B, 1))
ctx.step(u, n)
print("ok", ctx.counters()[1].mean(), ctx.profile(5), flush=True)
