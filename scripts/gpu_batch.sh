for bc in "64 16" "64 8" "64 4" "64 2" "128 4" "128 8"; do set -- $bc
timeout 300 python bench.py --steps 5 --warmup 3 --batch $1 --concurrency $2 --no-cpu-baseline > /tmp/b.json 2>&1; tail -1 /tmp/b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch', $1, 'conc', $2, 'value', round(d['value'],4), 'e2e', round(d['e2e']['value'],4), 'lat', round(d['latency_ms_per_image'],3), 'launches', d['gpu_launches'], d['config']['verified'])" || tail -3 /tmp/b.json
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | grep -E "^E |FAILED|passed|failed" | head -20
