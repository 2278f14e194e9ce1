mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gbc_smem -s 30 -c 1 -o gpurun_out/prof_gbc_smem2 python scripts/profile_config.py cifar_resnet18 1 > gpurun_out/ncu_gbc_smem2.log 2>&1; tail -1 gpurun_out/ncu_gbc_smem2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gbc_coef -s 30 -c 1 -o gpurun_out/prof_gbc_legacy2 env PC_GBC=0 python scripts/profile_config.py cifar_resnet18 1 > gpurun_out/ncu_gbc_legacy2.log 2>&1; tail -1 gpurun_out/ncu_gbc_legacy2.log
