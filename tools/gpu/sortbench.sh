# the default 50-step C5 bench (kernel-only) with a K2s re-sort every N steps (same box)
for r in 1 2; do
for N in ${NS:-0 24 32}; do
  ZPIC_SORT_EVERY=$N timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/sb_$N.log 2>&1
  python - $N <<'PY'
import json, sys
for l in open("gpurun_out/sb_%s.log" % sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l); k = d["kernel_ms_per_step"]
        print("every %3s  ms/step %.3f  value %.4g  K1 %.3f  sort %s  sm %s" % (sys.argv[1], d["ms_per_step"], d["value"], d["roofline"]["avg_launch_ms"], "%.2f" % k["k_sort_tiles"] if "k_sort_tiles" in k else "-", d["clocks"]["sm_mhz"]))
PY
done
done
