# Every config (kernel-only bench lines, per-kernel events and CUDA-graph replay), the tile sweep
# of the small / windowed configs and the weak-scaling mode at N = 1.  Output: gpurun_out/${TAG}_*.
TAG=${TAG:-cfg}
run() {   # label, bench args
  timeout 600 python bench.py --no-e2e --no-cpu "${@:2}" 2>&1 | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']
k = r['avg_launch_ms']
print('%-34s pushes/s %.3e ms/step %.4f K1 %s frac %s' % ('$1', d['value'], d['ms_per_step'], '%.4f' % k if k else '-', '%.3f' % r['frac'] if r['frac'] else '-'),
      {n: round(v, 4) for n, v in d['kernel_ms_per_step'].items() if v > 0.002})" >> gpurun_out/${TAG}_configs.log
}
rm -f gpurun_out/${TAG}_configs.log
for cfg in C1 C2 C3 C4 C5 P-WEIBEL P-LWFA P-COLD P-WARM; do
  extra=""
  case $cfg in P-WEIBEL|P-COLD|P-WARM) extra="--tile 8";; esac
  run "$cfg $extra" --steps ${STEPS:-20} --config $cfg $extra
  run "$cfg $extra --graphs" --steps ${STEPS:-20} --config $cfg $extra --graphs
done
for cfg in C2 C3 C4; do for t in 8 16 32; do
  run "$cfg tile $t --graphs" --steps ${STEPS:-20} --config $cfg --tile $t --graphs
done; done
for w in P-COLD P-WARM P-WEIBEL; do
  run "weak $w N=1" --steps ${STEPS:-20} --weak $w --tile 8
done
cat gpurun_out/${TAG}_configs.log
