# parity tests + a kernel-only bench line (no e2e / cpu legs)
set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
tail -n 15 gpurun_out/q_pytest.log
timeout 600 python bench.py --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/q_bench.log
python - <<'PY'
import json
for l in open("gpurun_out/q_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value %.4g  ms/step %.3f  frac %.3f  K1 %.3f ms" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["avg_launch_ms"]))
        print(d["kernel_ms_per_step"])
PY
tail -n 3 gpurun_out/q_bench.log
