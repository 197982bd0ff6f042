# K1 chunk-sorting variant every N steps (ZPIC_CSORT_EVERY): the 50-step workload and steady state
for N in ${NS:-0 1 2 4 8}; do
  for wk in "3 47" "100 20"; do
    set -- $wk
    ZPIC_CSORT_EVERY=$N timeout 900 python bench.py --no-e2e --no-cpu --warmup $1 --steps $2 > gpurun_out/cs.log 2>&1
    python - $N $1 <<'PY'
import json, sys
for l in open("gpurun_out/cs.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("csort %2s warmup %3s  ms/step %.3f  K1 %.3f  frac %.3f  sm %s" % (sys.argv[1], sys.argv[2], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["clocks"]["sm_mhz"]))
PY
  done
done
