"""Short scenarios for compute-sanitizer (SURVEY.md:291): every execution path of the substep on
C1 / C2-sized tanks, a few substeps each.  Usage:
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize.py [paths...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sph_inputs as si  # noqa: E402
from paper_2604_12505_b200 import SphContext  # noqa: E402

SCEN = {
    # name: (ell, B, kwargs, substeps)
    "coop_c1": (1.0, 1, dict(rebin_every=0, skin=0.15, exec_path=2), 12),
    "kernels_multikernel_c1": (1.0, 2, dict(rebin_every=0, skin=0.15, exec_path=1, rebuild_path=2), 6),
    "kernels_small_c1": (1.0, 3, dict(rebin_every=0, skin=0.15, exec_path=1, rebuild_path=1), 6),
    "kernels_small_c2": (4.0, 2, dict(rebin_every=0, skin=0.15, exec_path=1, rebuild_path=1), 3),
    "resident_c1": (1.0, 2, dict(rebin_every=0, skin=0.15, exec_path=3), 6),
    "resident_c2": (4.0, 2, dict(rebin_every=0, skin=0.15, exec_path=3), 3),
}


def run(name):
    ell, B, kw, n = SCEN[name]
    t = si.moving_tank(ell, seed=4, vel=0.05)
    kw = dict(kw)
    kw["skin"] = kw["skin"] * t.params.h
    ctx = SphContext(t.params, t.pv32(), t.ghost_b, n_rollouts=B, **kw)
    u = si.ensemble_inputs(list(range(B)), 2)[0] * 20.0
    ctx.step(u[:, 0], n)              # sph_step path (forced rebuilds inside: skin is small)
    y, _ = ctx.rollout(u[:, :1])      # graph / cooperative / resident tick path
    ctx.get_particles(B - 1)
    st = ctx.get_status()[0]
    ctx.close()
    print(f"{name}: status {st.tolist()} y0 {y[0, 0, :2]}", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(SCEN)
    for nm in names:
        run(nm)
