# K1's L2 and DRAM bytes per launch on the L2-resident configs (C1 / C2 fit in the
# 126 MB L2, so their K1 is bounded by L2, not HBM): one ncu pass per config, K1 after 3 steps.
set -x
for c in C1 C2 C3 C4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,lts__t_bytes.sum.per_second,lts__t_bytes.sum.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:k_push_tiles -s 3 -c 1 --csv --log-file gpurun_out/l2_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/l2_${c}_run.log 2>&1
done
