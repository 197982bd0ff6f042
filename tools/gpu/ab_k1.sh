# Same-box A/B of K1 variants (ordered: 3 warm-up steps; decayed: 100), kernel-only C5 lines.
# VARIANTS: "so:envassign ..." entries, e.g. "libzpic_b200.so:ZPIC_K1_SHAPE=4"; bit-identity of the
# first two .so on C2 and C4 (E, B, J, particles) first.
set -x
A=${BIT_A:-libzpic_b200.head.so}; B=${BIT_B:-libzpic_b200.so}
for cfg in C2 C4; do
  for v in $A $B; do ZPIC_SO=$v timeout 300 python tools/gpu/bitcmp.py $cfg 30 gpurun_out/bc_${cfg}_$v.npz > /dev/null 2>&1; done
  python tools/gpu/bitcmp.py --compare gpurun_out/bc_${cfg}_$A.npz gpurun_out/bc_${cfg}_$B.npz > gpurun_out/bc_cmp_$cfg.log 2>&1
done
rm -f gpurun_out/*.npz
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in ${VARIANTS}; do
    so=${v%%:*}; envs=""; [ "$so" != "$v" ] && envs=${v#*:}
    for wk in "3 10" "100 20"; do
      set -- $wk
      env ZPIC_SO=$so $envs timeout 600 python bench.py --no-e2e --no-cpu --warmup $1 --steps $2 > gpurun_out/abk.log 2>&1
      python - "$v" $1 <<'PY'
import json, sys
for l in open("gpurun_out/abk.log"):
    if l.startswith("{"):
        d = json.loads(l)
        k = d["kernel_ms_per_step"]
        print("%-40s warmup %3s  ms/step %.3f  K1 %.3f  frac %.3f  K3m %.3f  K4 %.3f  K5 %.3f  sm %s" % (sys.argv[1], sys.argv[2], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], k.get("k_mail_gather", 0), k.get("k_assemble_j", 0), k.get("k_yee", 0), d["clocks"]["sm_mhz"]))
PY
    done
  done
done
