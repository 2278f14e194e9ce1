# Round evidence: GPU tests, the default bench line, the launch list of one
# ResNet-34 verification and an ncu --set full capture of the conv kernel.
# usage (via gpurun): bash scripts/gpu/evidence.sh TAG
TAG=${1:-ev}
mkdir -p gpurun_out
bash scripts/gpu/check.sh $TAG
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3900 -c 4500 --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/one_image.py cifar_resnet34 1 > gpurun_out/launches_$TAG.log 2>&1
tail -2 gpurun_out/launches_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_gbc_flat" -s 150 -c 3 \
  -o gpurun_out/ncu_flat_$TAG python scripts/one_image.py cifar_resnet34 1 > gpurun_out/ncu_flat_$TAG.log 2>&1
tail -1 gpurun_out/ncu_flat_$TAG.log
