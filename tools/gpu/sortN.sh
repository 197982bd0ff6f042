# steady-state C5 step time with a K2s re-sort every N steps (ZPIC_SORT_EVERY), after W warm-up
# steps from injection; kernel-only lines over K timed steps
for N in ${NS:-0 8 16 32}; do
  ZPIC_SORT_EVERY=$N timeout 900 python bench.py --no-e2e --no-cpu --warmup ${W:-100} --steps ${K:-32} > gpurun_out/sort_$N.log 2>&1
  python - $N <<'PY'
import json, sys
for l in open("gpurun_out/sort_%s.log" % sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l); k = d["kernel_ms_per_step"]
        print("every %3s  ms/step %.3f  K1 %.3f  sort/launch %s  sm %s" % (sys.argv[1], d["ms_per_step"], d["roofline"]["avg_launch_ms"], "%.2f" % k["k_sort_tiles"] if "k_sort_tiles" in k else "-", d["clocks"]["sm_mhz"]))
PY
done
