for cfg in C3 C4 P-LWFA; do for t in 16 32; do
  timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --config $cfg --tile $t 2>&1 | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']
print('$cfg tile $t pushes/s %.3e ms/step %.4f K1 %.4f frac %.3f' % (d['value'], d['ms_per_step'], r['avg_launch_ms'], r['frac']))"
done; done
