# Same-box A/B of K5 tile shapes (libzpic_b200.yXXYY.so built with -DZPIC_YEE_TX / -DZPIC_YEE_TY)
for r in 1 2; do for v in ${VARIANTS:-y3232 y3216 y6416 y6432 y3264}; do
  for cfg in C5 C4; do
    ZPIC_SO=libzpic_b200.$v.so timeout 300 python bench.py --config $cfg --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); k = d['kernel_ms_per_step']
print('%-6s %-3s ms/step %.4f yee %.4f' % ('$v', '$cfg', d['ms_per_step'], k['k_yee']))"
  done
done; done
