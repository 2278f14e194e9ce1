mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q.json 2>/dev/null
tail -1 gpurun_out/q.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['latency_ms_per_image'],d['e2e']['value'],d['roofline']['kernel_ms'],d['roofline']['fp64']['frac'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_chk.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_chk.csv k_eval_layer at:: 2>/dev/null | head -12
