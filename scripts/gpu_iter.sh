# quick GPU iteration: parity tests + per-class profiles of the heavy configs
mkdir -p gpurun_out
python -m pytest tests/test_cpp_facade.py -q -m "not gpu" 2>&1 | tail -1
tests/cpp/build/test_facade 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5
for c in ${CONFIGS:-cifar_convbig cifar_resnet18 cifar_resnet34}; do
  timeout 900 python scripts/profile_config.py $c 1 2>&1 | tail -1 | cut -c1-1200
done
