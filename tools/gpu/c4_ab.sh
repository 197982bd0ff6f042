# Same-box A/B of the base library and the working tree on the windowed / filtered configs (C4,
# P-LWFA: the register filter and the window mailbox capacity) plus C3, and the bit-identity of
# C4 / P-LWFA / C1 after 40 steps (base twice: run-to-run determinism; the tree; the tree with
# the old filter).  Output: gpurun_out/${TAG:-ab}_c4.log
TAG=${TAG:-ab}
LOG=gpurun_out/${TAG}_c4.log
T=/tmp/bitcmp; mkdir -p $T
rm -f $LOG
for cfg in ${CFGS:-C4 P-LWFA C1}; do
  ZPIC_SO=libzpic_b200.base.so timeout 300 python tools/gpu/bitcmp.py $cfg 40 $T/${cfg}_base.npz >> $LOG 2>&1
  ZPIC_SO=libzpic_b200.base.so timeout 300 python tools/gpu/bitcmp.py $cfg 40 $T/${cfg}_base2.npz >> $LOG 2>&1
  timeout 300 python tools/gpu/bitcmp.py $cfg 40 $T/${cfg}_new.npz >> $LOG 2>&1
  ZPIC_FILTER_V1=1 timeout 300 python tools/gpu/bitcmp.py $cfg 40 $T/${cfg}_newv1.npz >> $LOG 2>&1
  for o in base2 new newv1; do
    echo "$cfg base vs $o:" >> $LOG
    python tools/gpu/bitcmp.py --compare $T/${cfg}_base.npz $T/${cfg}_$o.npz >> $LOG 2>&1
  done
done
for r in 1 2; do
  for cfg in ${TCFGS:-C4 P-LWFA}; do
    for v in libzpic_b200.base.so libzpic_b200.so; do
      for mode in "" "--graphs"; do
        ZPIC_SO=$v timeout 300 python bench.py --config $cfg $mode --no-cpu --no-e2e --steps 20 --warmup 5 2>/dev/null | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read())
k = {n: round(v, 4) for n, v in d.get('kernel_ms_per_step', {}).items() if v > 0.002}
print('%-6s %-22s %-8s ms/step %.4f' % ('$cfg', '$v', '$mode', d['ms_per_step']), k)" >> $LOG
      done
    done
  done
done
cat $LOG
