mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numeric.py -q -x 2>&1 | tail -2
run() { timeout 300 python bench.py --steps 5 --warmup 3 --batch 64 --concurrency 16 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', 'value', round(d['value'],3), 'lat', round(d['latency_ms_per_image'],3), 'dense_ms/launch', round(r['kernel_ms']/max(r['launches'],1),4), 'fp64frac', round(r['fp64']['frac'],3))"; }
run default
PC_BIG_CHAIN_CELLS=256 run big256
PC_EXEC_MODE=1 PC_LAZY_COMPACT=1 run lazy
