#!/usr/bin/env python3
"""Write the benchmark's settled start states with the float64 ORACLE (one-time, CPU):
damped settle (reading A17: v <- v exp(-10 dt) per substep, body pinned) of the lattice tank.
The bench loads these (float32) so its input does not depend on the CUDA path."""
import math, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O
import sph_inputs as si

def main(ell=4.0, seconds=6.0, out=None):
    t = si.make_tank(ell)
    sp = t.params
    s = O.State.from_tank(t)
    n = int(round(seconds / sp.dt)); chunk = int(round(0.5 / sp.dt))
    t0 = time.time()
    done = 0
    while done < n:
        m = min(chunk, n - done)
        s.step(n=m, damping=math.exp(-10 * sp.dt), pin_body=True)
        done += m
        print(f"t={done*sp.dt:5.2f}s max|v|={np.abs(s.vel).max():.3e} ({time.time()-t0:.0f}s)", flush=True)
    pv = np.concatenate([s.pos, s.vel], 1).astype(np.float32)
    out = out or os.path.join(ROOT, "bench_data", f"settled_ell{ell:g}.npz")
    np.savez_compressed(out, pv=pv, ell=ell, seconds=seconds, max_speed=float(np.abs(s.vel).max()),
                        recipe="oracle damped settle, reading A17, lattice start (sph_inputs.make_tank)")
    print("wrote", out)

if __name__ == "__main__":
    main(float(sys.argv[1]) if len(sys.argv) > 1 else 4.0, float(sys.argv[2]) if len(sys.argv) > 2 else 6.0)
