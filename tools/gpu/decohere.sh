# K1 in the ordered (freshly injected) vs decohered (after many steps) particle order:
# kernel-only C5 lines after 3 and after W warm-up steps, and ncu of K1 at 2048^2 after W steps
W=${W:-200}
for w in 3 $W; do
  timeout 900 python bench.py --no-e2e --no-cpu --warmup $w --steps 10 > gpurun_out/dec_$w.log 2>&1
  python - $w <<'PY'
import json, sys
for l in open("gpurun_out/dec_%s.log" % sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("warmup", sys.argv[1], "ms/step %.3f K1 %.3f frac %.3f" % (d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"]), d["clocks"])
PY
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_push_tiles -s $W -c 1 \
  -o gpurun_out/dec_k1 -f python bench.py --nx 2048 --ny 2048 --steps 2 --warmup $W --no-e2e --no-cpu > gpurun_out/dec_ncu.log 2>&1
ncu -i gpurun_out/dec_k1.ncu-rep --page source --csv --print-source sass > gpurun_out/dec_k1_source.csv 2>/dev/null
ncu -i gpurun_out/dec_k1.ncu-rep --page raw --csv > gpurun_out/dec_k1_raw.csv 2>/dev/null
