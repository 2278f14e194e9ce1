# compute-sanitizer runs over a parity subset (memcheck, racecheck, synccheck).
# usage (via gpurun): bash scripts/gpu/sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
SEL='tests/test_gpu_parity.py -k "(random_nets and 900) or batch_matches_sequential or golden_report or signed_zero"'
for tool in memcheck racecheck synccheck; do
  for mode in 1 2; do
    timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      env PC_EXEC_MODE=$mode python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
      -k "(random_nets and 900) or batch_matches_sequential or golden_report or signed_zero" \
      > gpurun_out/san_${TAG}_${tool}_mode$mode.txt 2>&1
    echo "$tool mode$mode rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_${TAG}_${tool}_mode$mode.txt | tail -3
  done
done
