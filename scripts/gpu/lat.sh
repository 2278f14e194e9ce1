# single-image latency of a config under engine switches (concurrent schedule)
# usage (via gpurun): bash scripts/gpu/lat.sh CONFIG "ENV1" "ENV2" ...
CFG=$1; shift
for env in "$@"; do
  echo "== $env"
  env $env PROBE_CONC_ONLY=1 timeout 600 python scripts/conv_probe.py $CFG 2>&1 | grep '"image": 1' | cut -c1-130
done
