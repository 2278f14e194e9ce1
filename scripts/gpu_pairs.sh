for p in 0 1; do
  PC_GBC_PAIRS=$p timeout 600 python scripts/profile_config.py cifar_resnet34 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pairs', $p, 'r34', d['device_ms'], d['classes']['gbc_coef'])"
  PC_GBC_PAIRS=$p timeout 600 python scripts/profile_config.py cifar_resnet18 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pairs', $p, 'r18', d['device_ms'], d['classes']['gbc_coef'])"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
