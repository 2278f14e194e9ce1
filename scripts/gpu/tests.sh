# GPU test suite only. usage (via gpurun): bash scripts/gpu/tests.sh TAG [pytest args]
TAG=${1:-t}; shift
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 "$@" > gpurun_out/pytest_$TAG.txt 2>&1; tail -25 gpurun_out/pytest_$TAG.txt
