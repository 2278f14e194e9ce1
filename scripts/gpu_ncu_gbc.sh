mkdir -p gpurun_out
for v in 1 0; do
PC_GBC=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:gbc -s 40 -c 4 -o gpurun_out/prof_gbc_v$v python scripts/profile_config.py cifar_resnet18 1 > gpurun_out/ncu_gbc_v$v.log 2>&1; tail -2 gpurun_out/ncu_gbc_v$v.log
done
