# K2s variants (ZPIC_SO) at C5: sort kernel time per launch, re-sort every 16 steps after 16 warm-up steps
for v in ${VARIANTS}; do
  ZPIC_SO=$v ZPIC_SORT_EVERY=16 timeout 600 python bench.py --no-e2e --no-cpu --warmup 16 --steps 32 > gpurun_out/sortab.log 2>&1
  python - $v <<'PY'
import json, sys
for l in open("gpurun_out/sortab.log"):
    if l.startswith("{"):
        d = json.loads(l); k = d["kernel_ms_per_step"]
        print("%-30s ms/step %.3f  K1 %.3f  sort %.2f ms  sm %s" % (sys.argv[1], d["ms_per_step"], d["roofline"]["avg_launch_ms"], k.get("k_sort_tiles", -1), d["clocks"]["sm_mhz"]))
PY
done
