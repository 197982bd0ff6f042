# tile size in both regimes (C5, kernel-only): steps 3-13 and 100-120
for T in ${TS:-8 16 32}; do
  for wk in "3 10" "100 20"; do
    set -- $wk
    timeout 600 python bench.py --no-e2e --no-cpu --tile $T --warmup $1 --steps $2 > gpurun_out/td.log 2>&1
    python - $T $1 <<'PY'
import json, sys
for l in open("gpurun_out/td.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("T %s warmup %3s  ms/step %.3f  K1 %.3f  frac %.3f  sm %s" % (sys.argv[1], sys.argv[2], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["clocks"]["sm_mhz"]))
PY
  done
done
