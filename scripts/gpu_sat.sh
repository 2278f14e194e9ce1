for bc in "512 8" "1024 16" "768 12" "512 4"; do
  set -- $bc
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --batch $1 --concurrency $2 > gpurun_out/bs.json 2>/dev/null
  echo "batch=$1 conc=$2 $(python -c "import json;d=json.loads(open('gpurun_out/bs.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])")"
done
