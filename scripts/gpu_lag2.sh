for lr in 0 64 100000 0; do
  PC_LAG_ROWS=$lr timeout 600 python scripts/profile_config.py cifar_resnet34 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag', $lr, 'r34', d['device_ms'], d['classes']['gbc_coef'])"
done
