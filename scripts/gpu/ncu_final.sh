# Round evidence: the launch list of one ResNet-34 verification (image 1,
# after the warm-up image) and ncu --set full captures of the conv kernel and
# of the prediction kernels.
# usage (via gpurun): bash scripts/gpu/ncu_final.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 8600 -c 9000 --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/one_image.py cifar_resnet34 1 > gpurun_out/launches_$TAG.log 2>&1
tail -2 gpurun_out/launches_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_gbc_flat" -s 150 -c 3 \
  -o gpurun_out/ncu_flat_$TAG python scripts/one_image.py cifar_resnet34 1 > gpurun_out/ncu_flat_$TAG.log 2>&1
tail -1 gpurun_out/ncu_flat_$TAG.log
timeout 900 ncu --set full --clock-control none -k "regex:k_pred_offer|k_pk_affine_terms|k_count_affine|k_affine_fold" -s 40 -c 8 \
  -o gpurun_out/ncu_pred_$TAG python scripts/one_image.py cifar_resnet34 1 > gpurun_out/ncu_pred_$TAG.log 2>&1
tail -1 gpurun_out/ncu_pred_$TAG.log
