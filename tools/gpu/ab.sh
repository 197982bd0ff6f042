# Same-box A/B timing of library variants: VARIANTS="libzpic_b200.so libzpic_b200.ab_x.so" (built
# in-tree), ROUNDS interleaved rounds of a kernel-only C5 bench line each.
for r in $(seq 1 ${ROUNDS:-3}); do
  for v in ${VARIANTS}; do
    ZPIC_SO=$v timeout 300 python bench.py --no-e2e --no-cpu --steps ${STEPS:-5} ${BENCH_ARGS} > gpurun_out/ab.log 2>&1
    python - $v $r <<'PY'
import json, sys
for l in open("gpurun_out/ab.log"):
    if l.startswith("{"):
        d = json.loads(l)
        k = d["kernel_ms_per_step"]
        print("%-28s round %s  ms/step %.3f  K1 %.3f ms  frac %.3f  | %s" % (sys.argv[1], sys.argv[2], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"],
              " ".join("%s %.3f" % (n[2:], v) for n, v in sorted(k.items()) if n != "k_push_tiles" and v > 0.05)))
PY
  done
done
