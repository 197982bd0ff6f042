# One ncu --set full capture of kernel $KREGEX (default k_yee) in the default C5 bench, source counters.
set -x
TAG=${TAG:-yee}
K=${KREGEX:-k_yee}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-2} -c 1 \
  -o gpurun_out/${TAG} -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
