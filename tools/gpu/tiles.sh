for cfg in C2 C3 C4 C5; do for t in 8 16; do
  timeout 600 python bench.py --no-e2e --no-cpu --steps 20 --config $cfg --tile $t 2>&1 | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']
print('$cfg tile $t pushes/s %.3e ms/step %.4f K1 %.4f frac %.3f' % (d['value'], d['ms_per_step'], r['avg_launch_ms'], r['frac']), {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items()})"
done; done
