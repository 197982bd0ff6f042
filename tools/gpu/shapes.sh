# K1 launch-shape sweep (ZPIC_K1_SHAPE: 0 = 256x3, 1 = 256x4, 2 = 128x6, 3 = 128x8), kernel-only bench lines
for sh in ${SHAPES:-0 1 2 3}; do
  ZPIC_K1_SHAPE=$sh timeout 300 python bench.py --no-e2e --no-cpu --steps 5 ${BENCH_ARGS} > gpurun_out/shape_$sh.log 2>&1
  python - $sh <<'PY'
import json, sys
for l in open("gpurun_out/shape_%s.log" % sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("shape", sys.argv[1], "value %.4g ms/step %.3f K1 %.3f ms frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"]))
PY
done
