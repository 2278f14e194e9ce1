mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for c in cifar_resnet18 cifar_resnet34; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -2 | cut -c1-900
done
