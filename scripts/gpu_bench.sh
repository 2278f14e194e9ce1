mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
sleep 2
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 2500 gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
for c in cifar_convbig cifar_resnet18; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --batch 16 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-700; done
