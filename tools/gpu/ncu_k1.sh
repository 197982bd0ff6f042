# One ncu --set full capture of K1 (k_push_tiles) at a 2048^2 C5-physics grid (67 M particles),
# source-level counters, plus the launch list of the default bench command.  Output: gpurun_out/
set -x
TAG=${TAG:-k1}
NX=${NX:-2048}
timeout 600 python bench.py --nx $NX --ny $NX --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_push_tiles -s 1 -c 1 \
  -o gpurun_out/${TAG} -f python bench.py --nx $NX --ny $NX --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ls -la gpurun_out
