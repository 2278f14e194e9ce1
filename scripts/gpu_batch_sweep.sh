# Batch size / worker-context sweep of the 9x500 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch" 2>&1 | tail -2
for bc in "512 8" "512 4" "1024 8" "256 2"; do
  set -- $bc
  timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --batch $1 --concurrency $2 > gpurun_out/bs.json 2>/dev/null
  echo "batch=$1 conc=$2 $(python -c "import json;d=json.loads(open('gpurun_out/bs.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'])")"
done
