"""Tick time of every execution path on a batch of tanks (diagnostic): ell, n_first, B."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import oracle as O
import sph_inputs as si
from paper_2604_12505_b200 import SphContext

ell = float(sys.argv[1]); nf = int(sys.argv[2]) or None; B = int(sys.argv[3])
paths = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 3]
t = si.make_tank(ell, n_first=nf) if nf else si.make_tank(ell)
sp = t.params
s = O.settle(t, seconds=1.0) if t.n_fluid < 2000 else None
pv = (np.concatenate([s.pos, s.vel], 1).astype(np.float32) if s is not None else
      np.ascontiguousarray(np.load(os.path.join(ROOT, "bench_data", "settled_ell4.npz"))["pv"], np.float32))
W, T = 2, 3
u = torch.from_numpy(si.ensemble_inputs(range(B), W + T)[0]).cuda()
for ex in paths:
    ctx = SphContext(sp, pv, t.ghost_b, n_rollouts=B, rebin_every=0, skin=0.15 * sp.h, exec_path=ex)
    ctx.rollout(u[:, :W].contiguous())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    ctx.rollout(u[:, W:].contiguous())
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / T
    print(f"ell={ell} N={t.n_fluid} B={B} exec={ctx.exec_path()}: {ms:.3f} ms/tick "
          f"{B * t.n_fluid * sp.n_sub / ms / 1e6:.2f} G/s status {int(ctx.get_status()[0].max())}", flush=True)
    ctx.close()
