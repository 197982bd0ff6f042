# ncu --set full of K2s (k_sort_tiles) at C5 after 16 steps
timeout 1200 env ZPIC_SORT_EVERY=16 ncu --set full --clock-control none --import-source on -k regex:k_sort_tiles -c 1 \
  -o gpurun_out/sort_k2s -f python bench.py --steps 2 --warmup 16 --no-e2e --no-cpu > gpurun_out/sort_ncu.log 2>&1
ncu -i gpurun_out/sort_k2s.ncu-rep --page raw --csv > gpurun_out/sort_k2s_raw.csv 2>/dev/null
ncu -i gpurun_out/sort_k2s.ncu-rep --page source --csv --print-source sass > gpurun_out/sort_k2s_source.csv 2>/dev/null
