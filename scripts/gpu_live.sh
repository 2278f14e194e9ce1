# Live-column dense kernels: parity, bench, launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
for v in "PC_DENSE_LIVE=1" "PC_DENSE_LIVE=0" "PC_DENSE_LIVE=1 PC_DENSE_TM=8"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/lv.json 2>/dev/null
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/lv.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['latency_ms_per_image'])")"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_live.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_live.csv k_eval_layer at:: 2>/dev/null | head -12
