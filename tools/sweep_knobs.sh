run() { # label env... args
  lbl=$1; shift
  env "$@" timeout 200 python bench.py --no-cpu-baseline $ARGS 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lbl', round(d['value']/1e9,3), {k: round(v*1000,1) for k,v in d['roofline']['live_ms'].items()})" >> gpurun_out/sweep2.log 2>&1
}
for r in 1 2; do
ARGS=""; run base X=1
ARGS="--skin 0.14"; run skin0.14 X=1
ARGS="--skin 0.17"; run skin0.17 X=1
ARGS=""; run pf1 SPH_PF=1
ARGS=""; run pf2 SPH_PF=2
ARGS=""; run dtile64 SPH_DTILE=64
ARGS=""; run ntile64 SPH_NTILE=64
ARGS=""; run ntile256 SPH_NTILE=256
done
