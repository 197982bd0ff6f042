# Round profile artefacts (summaries are copied into profiles/ afterwards):
#  1. default bench line;  2. ncu launch list of bench --steps 2 --warmup 1 (C5);
#  3. K1 DRAM bytes per launch at C5 (2 metrics, one pass);  4. ncu --set full of K1 at 2048^2.
set -x
TAG=${TAG:-pr}
[ -f gpurun_out/${TAG}_bench.log ] || timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_launches_run.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_push_tiles -s 2 -c 1 --csv --log-file gpurun_out/${TAG}_traffic.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_traffic_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push_tiles -s 1 -c 1 \
  -o gpurun_out/${TAG}_k1 -f python bench.py --nx 2048 --ny 2048 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_k1_run.log 2>&1
ncu -i gpurun_out/${TAG}_k1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_k1_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_k1.ncu-rep --page raw --csv > gpurun_out/${TAG}_k1_raw.csv 2>/dev/null
ls -la gpurun_out
