# Same-box A/B of K3m (k_mail_gather) launch-bound variants at C5: per-kernel event times
for r in 1 2; do for v in ${VARIANTS:-base k3m4 k3m6 k3m8}; do
  ZPIC_SO=libzpic_b200.$v.so timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); k = d['kernel_ms_per_step']
print('%-8s ms/step %.3f K1 %.3f K3m %.4f K3 %.4f' % ('$v', d['ms_per_step'], k['k_push_tiles'], k['k_mail_gather'], k['k_insert']))"
done; done
