# ncu --set full of k_gbc_flat launches inside one refinement pass of
# ResNet-34 (NVTX range "pass T"; pass 37 is the 237-row pass that dominates
# the image), image 0 only, summarised on the box.
# usage (via gpurun): bash scripts/gpu/ncu_flat.sh TAG [PASS] [SKIP] [COUNT]
TAG=${1:-flat}; PASS=${2:-37}; SKIP=${3:-10}; CNT=${4:-6}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "pass $PASS/" \
  -k "regex:k_gbc_flat" -s $SKIP -c $CNT \
  -o gpurun_out/ncu_flat_$TAG python scripts/one_image.py cifar_resnet34 0 > gpurun_out/ncu_flat_$TAG.log 2>&1
tail -1 gpurun_out/ncu_flat_$TAG.log
python scripts/ncu_summary.py gpurun_out/ncu_flat_$TAG.ncu-rep > gpurun_out/ncu_flat_$TAG.txt 2>&1
# keep the report small enough to travel back (gpurun merges <= 64 MiB)
[ $(stat -c %s gpurun_out/ncu_flat_$TAG.ncu-rep) -gt 40000000 ] && rm -f gpurun_out/ncu_flat_$TAG.ncu-rep
