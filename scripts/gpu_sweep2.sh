for v in "PC_GBC_MINB=2 PC_GBC_L1=1" "PC_GBC_MINB=3 PC_GBC_L1=1" "PC_GBC_MINB=4 PC_GBC_L1=1" "PC_GBC_MINB=2 PC_GBC_L1=0" "PC_GBC_MINB=3 PC_GBC_L1=1"; do
  env $v timeout 600 python scripts/profile_config.py cifar_resnet34 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'r34', d['device_ms'])"
done
