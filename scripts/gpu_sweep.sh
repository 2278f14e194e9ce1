for c in 1 4 8 16 32; do
  timeout 300 python bench.py --steps 5 --warmup 3 --batch 64 --concurrency $c --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conc', $c, 'value', round(d['value'],3), 'lat', round(d['latency_ms_per_image'],3), 'launches', d['gpu_launches'], d['roofline']['fp64'])"
done
