timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_sharding.py -q -x 2>&1 | tail -2
for lr in 0 64 100000; do
  PC_LAG_ROWS=$lr timeout 600 python scripts/profile_config.py cifar_resnet34 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag', $lr, 'r34', d['device_ms'], d['classes']['gbc_coef'])"
  PC_LAG_ROWS=$lr timeout 600 python scripts/profile_config.py mnist_9x500 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag', $lr, '9x500', d['device_ms'])"
done
