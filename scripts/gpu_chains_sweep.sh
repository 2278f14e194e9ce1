# Chain-kernel choice for batched walks, 9x500 and conv configs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cs.json 2>/dev/null
echo "9x500 default $(python -c "import json;d=json.loads(open('gpurun_out/cs.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['latency_ms_per_image'])")"
for c in cifar_convbig cifar_resnet18; do
for v in 256 4096 1000000000; do
  PC_BIG_CHAIN_CELLS_BATCHED=$v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --batch 16 --no-cpu-baseline > gpurun_out/cs.json 2>/dev/null
  echo "$c batched_big_from=$v $(python -c "import json;d=json.loads(open('gpurun_out/cs.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])")"
done
done
