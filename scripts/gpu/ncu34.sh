# ncu evidence for the ResNet-34 headline: the launch list of one verification
# (after a warm-up image) and full captures of the top kernels.
# usage (via gpurun): bash scripts/gpu/ncu34.sh TAG [kernel-regex] [skip]
TAG=${1:-ncu}
RX=${2:-"k_chain_affine_big|k_concretize_big|k_chain_relu_big|k_gbc_live|k_relu_coef|k_merge|k_compact_cells"}
SKIP=${3:-4000}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3900 -c 4200 --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/one_image.py cifar_resnet34 1 > gpurun_out/launches_$TAG.log 2>&1
tail -2 gpurun_out/launches_$TAG.log
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$RX" -s $SKIP -c 14 \
  -o gpurun_out/prof_$TAG python scripts/one_image.py cifar_resnet34 1 > gpurun_out/prof_$TAG.log 2>&1
tail -3 gpurun_out/prof_$TAG.log
ls -la gpurun_out/
