# median single-image latency of a config under engine switches
# usage (via gpurun): bash scripts/gpu/latsmall.sh CONFIG N "ENV1" "ENV2" ...
CFG=$1; N=$2; shift 2
for env in "$@"; do
  echo "== $env"
  env $env timeout 600 python scripts/latency.py $CFG $N 2>&1 | tail -1
done
