# precision experiment: one-word int32 current (default) vs the exact two-word form (ZPIC_FX_SMIN=99)
for smin in 22 99; do
  ZPIC_FX_SMIN=$smin timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "paper_weibel or c1_full or c2_weibel" -s 2>&1 | grep -E "^\{|passed|failed|Error" | cut -c1-400 | sed "s/^/SMIN=$smin /"
done
