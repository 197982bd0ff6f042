# new parity tests + NEXT-3 / NEXT-4 bench lines (kernel-only)
set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "commutative or paper or c1_full" -s > gpurun_out/n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n_pytest.log
tail -n 5 gpurun_out/n_pytest.log
for args in "--current-mode 1" "--config P-WEIBEL --tile 8" "--config P-WEIBEL --tile 16" "--config P-LWFA" "--config P-WARM --tile 8" "--config C2" "--config C3" "--config C4"; do
  timeout 600 python bench.py --no-e2e --no-cpu --steps 10 $args > gpurun_out/n_bench.tmp 2>&1
  echo "ARGS $args" >> gpurun_out/n_bench.log; cat gpurun_out/n_bench.tmp >> gpurun_out/n_bench.log
done
python - <<'PY'
import json
args = None
for l in open("gpurun_out/n_bench.log"):
    if l.startswith("ARGS"): args = l.strip()
    if l.startswith("{"):
        d = json.loads(l)
        print(args, "| value %.4g  ms/step %.3f  K1 %.3f ms frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"]), {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()})
PY
