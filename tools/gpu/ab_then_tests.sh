# same-box A/B of a K1 variant against the previous build, then the GPU test suite on the new one
BIT_A=${BIT_A:-libzpic_b200.prev.so} BIT_B=libzpic_b200.so VARIANTS="${VARIANTS:-libzpic_b200.prev.so libzpic_b200.so}" ROUNDS=${ROUNDS:-3} \
  bash tools/gpu/ab_k1.sh > gpurun_out/ab_new.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
