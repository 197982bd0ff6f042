# K1 L2 bulk-prefetch distance sweep (ZPIC_K1_PF chunks ahead; 0 = off), kernel-only C5 lines
for pf in ${PFS:-0 1 2 3 4}; do
  ZPIC_K1_PF=$pf timeout 300 python bench.py --no-e2e --no-cpu --steps 5 ${BENCH_ARGS} > gpurun_out/pf_$pf.log 2>&1
  python - $pf <<'PY'
import json, sys
for l in open("gpurun_out/pf_%s.log" % sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("pf", sys.argv[1], "value %.4g ms/step %.3f K1 %.3f ms frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"]))
PY
done
