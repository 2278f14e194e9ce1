mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gbc --csv --log-file gpurun_out/launches_r34_gbc.csv python scripts/profile_config.py cifar_resnet34 1 > gpurun_out/ncu_r34.log 2>&1; tail -2 gpurun_out/ncu_r34.log
