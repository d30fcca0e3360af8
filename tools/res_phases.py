"""Summarise SPH_RES_TIMING phase stamps: per phase, the mean over substeps of the slowest and the
median CTA's duration (us).  Phases: 0 start, 1 after rebuild, 2 after density, 3 after barrier A,
4 after aux pull + forces, 5 after barrier B, 6 after pv pull + body step, 7 after ghosts."""
import sys
import numpy as np
raw = np.fromfile(sys.argv[1], dtype=np.uint64)
off = 0
launches = []
while off < raw.size:
    n, ns = int(raw[off]), int(raw[off + 1])
    a = raw[off + 2: off + 2 + n * ns * 8].reshape(n, ns, 8).astype(np.int64)
    launches.append(a)
    off += 2 + n * ns * 8
a = launches[-1]
names = ["rebuild", "density", "barrier A", "aux pull+force", "barrier B", "pv pull+body", "ghosts", "(next)"]
ok = (a > 0).all(axis=2)
d = np.diff(a, axis=2)        # [cta, substep, 7]
for k in range(7):
    v = d[:, :, k][ok[:, :]].reshape(-1) if False else d[:, :, k]
    print(f"{names[k]:16s} median-CTA {np.median(v) / 1e3:7.3f} us   slowest-CTA mean {np.mean(v.max(axis=0)) / 1e3:7.3f} us")
tot = (a[:, :, 7] - a[:, :, 0])
print(f"substep (CTA 0) mean {np.mean(tot[0]) / 1e3:.3f} us over {a.shape[1]} substeps, {a.shape[0]} CTAs")
