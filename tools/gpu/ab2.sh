# Same-box A/B of library variants in both regimes: ordered (steps 3-13 after the injection) and
# decayed (steps 100-120); kernel-only C5 lines
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in ${VARIANTS}; do
    for wk in "3 10" "100 20"; do
      set -- $wk
      ZPIC_SO=$v timeout 600 python bench.py --no-e2e --no-cpu --warmup $1 --steps $2 > gpurun_out/ab2.log 2>&1
      python - $v $1 <<'PY'
import json, sys
for l in open("gpurun_out/ab2.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("%-28s warmup %3s  ms/step %.3f  K1 %.3f  frac %.3f  sm %s" % (sys.argv[1], sys.argv[2], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["clocks"]["sm_mhz"]))
PY
    done
  done
done
