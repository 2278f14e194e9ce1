for v in "PC_GBC=0" "PC_GBC_PW=1" "PC_GBC_PW=2" "PC_GBC_PW=4" "PC_GBC_PW=8" "X=1"; do
  env $v timeout 600 python scripts/profile_config.py cifar_resnet18 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'device_ms', d['device_ms'], 'gbc', d['classes'].get('gbc_coef'))"
done
env PC_GBC=0 timeout 900 python scripts/profile_config.py cifar_resnet34 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r34 legacy', 'device_ms', d['device_ms'], 'gbc', d['classes'].get('gbc_coef'))"
