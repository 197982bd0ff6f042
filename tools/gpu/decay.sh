# K1 time vs steps since the (ordered) injection: kernel-only C5 lines after W warm-up steps
for w in ${WS:-3 10 20 40 100}; do
  timeout 900 python bench.py --no-e2e --no-cpu --warmup $w --steps 5 > gpurun_out/decay_$w.log 2>&1
  python - $w <<'PY'
import json, sys
for l in open("gpurun_out/decay_%s.log" % sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("warmup %4s  ms/step %.3f  K1 %.3f  frac %.3f  sm %s" % (sys.argv[1], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["clocks"]["sm_mhz"]))
PY
done
