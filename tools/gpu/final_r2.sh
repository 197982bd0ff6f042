TAG=r2w bash tools/gpu/profile_all.sh > gpurun_out/pa.log 2>&1
W=200 bash tools/gpu/decohere.sh > gpurun_out/dec.log 2>&1
bash tools/gpu/l2_small.sh > gpurun_out/l2.log 2>&1
