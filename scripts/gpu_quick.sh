mkdir -p gpurun_out
PC_EXEC_MODE=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for m in 1 2; do for c in 16; do
PC_EXEC_MODE=$m timeout 300 python bench.py --steps 5 --warmup 3 --batch 64 --concurrency $c --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode', $m, 'conc', $c, 'value', round(d['value'],3), 'lat', round(d['latency_ms_per_image'],3))"
done; done
