# quick GPU iteration: parity tests + per-class profiles of the heavy configs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv,noheader
for c in ${CONFIGS:-cifar_convbig cifar_resnet18 cifar_resnet34}; do
  timeout 900 python scripts/profile_config.py $c ${NIMG:-1} 2>&1 | tail -${NIMG:-1} | cut -c1-1200
done
