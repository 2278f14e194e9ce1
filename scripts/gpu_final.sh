# Round-end evidence: bench lines, launch list, ncu captures, per-class profiles, tests.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 3000 gpurun_out/bench_final.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_final.json 2>&1; tail -c 1200 gpurun_out/bench_ref_final.json
for c in cifar_convbig cifar_resnet18; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --batch 16 --no-cpu-baseline > gpurun_out/bench_final_$c.json 2>&1; tail -c 600 gpurun_out/bench_final_$c.json
done
for c in mnist_6x100 cifar_convbig cifar_resnet18 cifar_resnet34; do
  timeout 900 python scripts/profile_config.py $c 2 > gpurun_out/prof_final_$c.jsonl 2>&1; tail -1 gpurun_out/prof_final_$c.jsonl | cut -c1-300
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
PYTHONPATH=. timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_coef3 -s 20 -c 2 -o gpurun_out/prof_dense3_final python scripts/one_batch.py > /dev/null 2>&1
PYTHONPATH=. timeout 900 ncu --metrics sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/met_final.csv python scripts/one_batch.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gbc_sparse -s 30 -c 2 -o gpurun_out/prof_gbc_sparse_final python scripts/profile_config.py cifar_resnet18 1 > /dev/null 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
ls gpurun_out
