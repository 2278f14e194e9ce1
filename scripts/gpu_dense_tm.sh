# Dense coefficient kernel variants on the batched bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch or mnist" 2>&1 | tail -2
for v in "PC_DENSE_V2=0 PC_DENSE_TM=4" "PC_DENSE_V2=1 PC_DENSE_TM=4" "PC_DENSE_V2=1 PC_DENSE_TM=8" "PC_DENSE_V2=1 PC_DENSE_TM=3" "PC_DENSE_V2=1 PC_DENSE_TM=0" "PC_DENSE_V2=0 PC_DENSE_TM=4"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tm.json 2>/dev/null
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/tm.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['fp64']['frac'])")"
done
PC_DENSE_TM=4 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tm.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_tm.csv k_eval_layer at:: 2>/dev/null | head -6
PC_DENSE_TM=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dense_coef2 -s 40 -c 1 -o gpurun_out/ncu_b_dense2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
