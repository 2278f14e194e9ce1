mkdir -p gpurun_out
python scripts/dbg_band.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gbc_smem -s 20 -c 2 -o gpurun_out/prof_gbc_smem python scripts/profile_config.py cifar_resnet18 1 > gpurun_out/ncu_gbc_smem.log 2>&1; tail -2 gpurun_out/ncu_gbc_smem.log
