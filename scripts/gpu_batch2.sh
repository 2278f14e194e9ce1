for bc in "128 4" "128 2" "256 4" "256 8" "192 6"; do set -- $bc
timeout 300 python bench.py --steps 5 --warmup 3 --batch $1 --concurrency $2 --no-cpu-baseline > /tmp/b.json 2>&1; tail -1 /tmp/b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch', $1, 'conc', $2, 'value', round(d['value'],4), 'fp64', round(d['roofline']['fp64']['frac'],3))" || tail -3 /tmp/b.json
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x 2>&1 | tail -1
