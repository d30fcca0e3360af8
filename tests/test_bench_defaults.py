"""The measured configuration of bench.py is entirely in its arguments (no environment knobs):
pin the per-workload defaults the driver's plain `python bench.py` runs with (DESIGN.md §7c,
r02.36 / r02.43) and the documented override rules.  CPU only; imports nothing GPU-side."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _resolve(*argv):
    b = _bench()
    return b.resolve_defaults(b.parse(list(argv)))


def test_default_line_is_c3_with_the_adaptive_skin():
    a = _resolve()
    assert a.workload == "C3" and a.gpus == 1 and a.steps == 10 and a.warmup >= 3
    assert (a.skin, a.skin_max, a.skin_mode) == (0.10, 0.7, 0)   # B5 0.10h -> 0.7h
    assert a.impl == "ours"


def test_workload_skin_policies():
    a = _resolve("--workload", "C5")
    assert (a.skin, a.skin_max, a.skin_mode) == (0.10, 0.7, 0)
    a = _resolve("--workload", "C4")
    assert (a.skin, a.skin_max, a.skin_mode) == (0.15, 0.8, 1)     # B6 half-skins
    assert abs(a.settle_seconds - 1e-3 * 1000 / 42.0) < 1e-15
    a = _resolve("--workload", "P0")
    assert (a.skin, a.skin_max) == (0.5, 0.0)                      # fixed skin (B4)


def test_explicit_skin_alone_is_a_fixed_skin_and_overrides_compose():
    a = _resolve("--skin", "0.2")
    assert (a.skin, a.skin_max) == (0.2, 0.0)
    a = _resolve("--skin", "0.12", "--skin-max", "0.5")
    assert (a.skin, a.skin_max) == (0.12, 0.5)
