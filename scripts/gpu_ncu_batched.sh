# ncu --set full of the top kernels of the batched 9x500 bench step.
mkdir -p gpurun_out
for k in k_dense_coef k_fwd_dense k_concretize_big k_chain_affine_big; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 2 -o gpurun_out/ncu_b_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out/*.ncu-rep
