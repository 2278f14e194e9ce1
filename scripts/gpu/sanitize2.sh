# compute-sanitizer over the round-2 paths: the parity subset (host-driven
# schedule: predicted compaction, fused partials, device-applied compaction)
# and whole verifications of ConvBig / ResNet-18 (staged forward conv, the
# live-cell conv kernel, the prediction kernels at real sizes).
# usage (via gpurun): bash scripts/gpu/sanitize2.sh TAG
TAG=${1:-san2}
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
  -k "(random_nets and 900) or batch_matches_sequential or golden_report or signed_zero" \
  > gpurun_out/san_${TAG}_memcheck_parity.txt 2>&1
echo "memcheck parity rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_${TAG}_memcheck_parity.txt | tail -3
for cfg in cifar_convbig cifar_resnet18; do
  for tool in memcheck racecheck synccheck; do
    [ "$cfg" = cifar_resnet18 ] && [ "$tool" != memcheck ] && continue
    ONE_IMAGE_FIRST=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 20 \
      python scripts/one_image.py $cfg 1 > gpurun_out/san_${TAG}_${tool}_$cfg.txt 2>&1
    echo "$tool $cfg rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|True|False" gpurun_out/san_${TAG}_${tool}_$cfg.txt | tail -3
  done
done
