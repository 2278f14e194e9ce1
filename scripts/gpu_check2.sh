mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x -k "dense" 2>&1 | tail -1
for r in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q.json 2>/dev/null
tail -1 gpurun_out/q.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['latency_ms_per_image'],d['e2e']['value'],d['roofline']['kernel_ms'],d['roofline']['fp64']['frac'])"
done
PYTHONPATH=. timeout 900 ncu --metrics sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/met_chk.csv python scripts/one_batch.py > /dev/null 2>&1
python scripts/sum_metrics.py gpurun_out/met_chk.csv > gpurun_out/met_chk.txt; head -4 gpurun_out/met_chk.txt; tail -1 gpurun_out/met_chk.txt
