# GPU check: build state, smoke, the GPU test suite, the default bench line.
# usage (from the repo root, via gpurun): bash scripts/gpu/check.sh TAG
TAG=${1:-check}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_$TAG.txt 2>&1; tail -25 gpurun_out/pytest_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 4000 gpurun_out/bench_$TAG.json; tail -5 gpurun_out/bench_$TAG.err
