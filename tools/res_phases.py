"""Summarise SPH_RES_TIMING phase stamps (diagnostic build, see RES_MARK in sph_resident.cuh): per
phase, the median CTA's and the mean over substeps of the slowest CTA's duration (us), and the
per-CTA means of the density and force phases.  File: records of [header CTAs, n_sub, marks]
followed by [CTAs][n_sub][marks] uint64 ns; the last launch is summarised."""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64)
off = 0
launches = []
while off < raw.size:
    n, ns, nm = int(raw[off]), int(raw[off + 1]), int(raw[off + 2])
    launches.append(raw[off + 3: off + 3 + n * ns * nm].reshape(n, ns, nm).astype(np.int64))
    off += 3 + n * ns * nm
a = launches[-1]
names = ["rebuild", "density", "barrier A", "aux pull+force", "barrier B", "partial loads (w0)",
         "warp reduce (w0)", "body update (l0)", "pv pull / sync", "ghosts"]
# substeps where every stamp was written (the last may break early)
ok = (a > 0).all(axis=(0, 2))
a = a[:, ok]
d = np.diff(a, axis=2)        # [cta, substep, marks - 1]
for k in range(d.shape[2]):
    v = d[:, :, k]
    print(f"{names[k]:20s} median-CTA {np.median(v) / 1e3:7.3f} us   slowest-CTA mean {np.mean(v.max(axis=0)) / 1e3:7.3f} us")
tot = a[:, :, -1] - a[:, :, 0]
print(f"substep (CTA 0) mean {np.mean(tot[0]) / 1e3:.3f} us over {a.shape[1]} substeps, {a.shape[0]} CTAs")
print("per-CTA density us", np.round(d[:, :, 1].mean(1) / 1e3, 2))
print("per-CTA force us  ", np.round(d[:, :, 3].mean(1) / 1e3, 2))
