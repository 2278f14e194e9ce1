# Iteration check: GPU tests, ResNet-34 class profile, short latency bench.
# usage (via gpurun): bash scripts/gpu/iter.sh TAG [skip-tests]
TAG=${1:-it}
mkdir -p gpurun_out
if [ "$2" != "skip-tests" ]; then
  timeout 1800 python -m pytest ${PYTEST_SEL:-tests} -m gpu -q -x --durations=8 --timeout 900 > gpurun_out/pytest_$TAG.txt 2>&1; tail -12 gpurun_out/pytest_$TAG.txt
fi
timeout 600 python scripts/profile_config.py cifar_resnet34 2 > gpurun_out/prof34_$TAG.jsonl 2>&1; cut -c1-1500 gpurun_out/prof34_$TAG.jsonl
timeout 900 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --throughput-images 0 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ["value","e2e","parity","verified","gpu_launches"]})
print(d["roofline"]["frac"], d["roofline"]["fp64_pipe_frac"], d["roofline"]["kernel_ms"])
PY
tail -3 gpurun_out/bench_$TAG.err
