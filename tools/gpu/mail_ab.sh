for cfg in C3 C4 C5; do for m in 0 1; do
  ZPIC_MAIL=$m timeout 600 python bench.py --no-e2e --no-cpu --steps 20 --config $cfg 2>&1 | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); k = d['kernel_ms_per_step']
print('$cfg mail=$m ms/step %.4f K1 %.4f K3 %.4f K3m %.4f' % (d['ms_per_step'], k['k_push_tiles'], k.get('k_insert', 0), k.get('k_mail_gather', 0)))"
done; done
