for p in 1 2; do
  PC_PIPES=$p timeout 600 python scripts/profile_config.py cifar_resnet34 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipes', $p, 'r34', d['device_ms'])"
  PC_PIPES=$p timeout 600 python scripts/profile_config.py cifar_resnet18 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipes', $p, 'r18', d['device_ms'])"
  PC_PIPES=$p timeout 600 python scripts/profile_config.py cifar_convbig 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipes', $p, 'convbig', d['device_ms'])"
  PC_PIPES=$p timeout 600 python scripts/profile_config.py mnist_9x500 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipes', $p, '9x500', d['device_ms'])"
  PC_PIPES=$p timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipes', $p, 'bench value', round(d['value'],3), 'lat', round(d['latency_ms_per_image'],3))"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_sharding.py -q -x 2>&1 | tail -2
