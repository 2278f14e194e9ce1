# quick conv / latency probes. usage (via gpurun): bash scripts/gpu/probe.sh TAG "ENV1" "ENV2" ...
TAG=${1:-probe}; shift
mkdir -p gpurun_out
for env in "$@"; do
  echo "== $env"
  env PROBE_SERIAL_ONLY=1 $env timeout 600 python scripts/conv_probe.py cifar_resnet34 2>&1 | tee -a gpurun_out/probe_$TAG.txt | tail -1 | cut -c1-300
done
