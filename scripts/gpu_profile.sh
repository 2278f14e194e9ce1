mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for c in mnist_9x500 cifar_convbig cifar_resnet18 cifar_resnet34; do
  timeout 600 python scripts/profile_config.py $c 1 2>&1 | tail -2
done
