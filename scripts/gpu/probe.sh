# quick conv / latency probes. usage (via gpurun): bash scripts/gpu/probe.sh TAG
TAG=${1:-probe}
mkdir -p gpurun_out
for env in "" "PC_LIVE_CELLS=0" "PC_LAZY_COMPACT=1" "PC_PIPES=1"; do
  echo "== $env"
  env $env timeout 600 python scripts/conv_probe.py cifar_resnet34 2>&1 | tee -a gpurun_out/probe_$TAG.txt | cut -c1-400
done
