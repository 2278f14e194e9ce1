run() { python bench.py --steps 10 --warmup 3 --batch 64 --concurrency 16 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'ms_per_step', round(d['ms_per_step'],1), d['clocks'])"; }
nproc
run
echo two processes:
run & run & wait
