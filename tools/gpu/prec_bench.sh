for smin in 22 99; do
  for args in "" "--config C3" "--config P-WARM --tile 8"; do
    ZPIC_FX_SMIN=$smin timeout 600 python bench.py --no-e2e --no-cpu --steps 5 $args 2>&1 | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('SMIN=$smin', '$args', 'K1 %.3f ms step %.3f ms frac %.3f' % (d['roofline']['avg_launch_ms'], d['ms_per_step'], d['roofline']['frac']))"
  done
done
