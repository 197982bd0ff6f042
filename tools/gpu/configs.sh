# every config, kernel-only bench lines, with and without CUDA-graph replay
set -x
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_pytest.log
tail -n 3 gpurun_out/c_pytest.log
rm -f gpurun_out/c_bench.log
for cfg in C1 C2 C3 C4 C5 P-WEIBEL P-LWFA P-COLD P-WARM; do
  for g in "" "--graphs"; do
    extra=""
    case $cfg in P-WEIBEL|P-COLD|P-WARM) extra="--tile 8";; esac
    timeout 600 python bench.py --no-e2e --no-cpu --steps ${STEPS:-20} --config $cfg $extra $g > gpurun_out/c_tmp.log 2>&1
    echo "ARGS $cfg $extra $g" >> gpurun_out/c_bench.log; grep "^{" gpurun_out/c_tmp.log >> gpurun_out/c_bench.log
  done
done
python - <<'PY'
import json
args = None
for l in open("gpurun_out/c_bench.log"):
    if l.startswith("ARGS"): args = l.strip()[5:]
    elif l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print("%-28s pushes/s %.3e  ms/step %.4f  K1 %s frac %s launches/step %.1f" % (args, d["value"], d["ms_per_step"],
              "%.4f" % r["avg_launch_ms"] if r["avg_launch_ms"] else "-", "%.3f" % r["frac"] if r["frac"] else "-", d["gpu_launches"] / d["steps"]))
PY
