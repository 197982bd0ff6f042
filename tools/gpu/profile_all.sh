# round profile artefacts (TAG prefix): validation, bench line, launch list, K1 traffic at C5,
# ncu --set full of K1 (2048^2) and of the other step kernels at C5
set -x
TAG=${TAG:-r1c}
bash tools/gpu/validate.sh
cp gpurun_out/bench.log gpurun_out/${TAG}_bench.log
TAG=$TAG bash tools/gpu/profile_round.sh
for k in k_yee k_mail_gather k_assemble_j; do
  TAG=${TAG}_$k KREGEX=$k bash tools/gpu/ncu_kernel.sh
done
ls gpurun_out
