# Parity + variants + bench (9x500 batched, latency) check.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q.json 2>/dev/null
tail -1 gpurun_out/q.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['latency_ms_per_image'],d['e2e']['value'],d['roofline']['fp64'])"
