mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for c in mnist_6x100 mnist_9x500 cifar_convbig; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value', round(d['value'],3), 'e2e', round(d['e2e']['value'],3), 'lat', d['latency_ms_per_image'], 'launches', d['gpu_launches'], d['config']['verified'], d['clocks'])"
done
