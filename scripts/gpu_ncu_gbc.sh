mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gbc_coef -s 40 -c 3 -o gpurun_out/prof_gbc_band python scripts/profile_config.py cifar_resnet18 1 > gpurun_out/ncu_gbc_band.log 2>&1; tail -2 gpurun_out/ncu_gbc_band.log
