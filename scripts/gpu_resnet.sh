mkdir -p gpurun_out
for c in cifar_resnet18 cifar_resnet34; do
  timeout 900 python scripts/profile_config.py $c 2 > gpurun_out/prof_$c.jsonl 2>&1; tail -c 2500 gpurun_out/prof_$c.jsonl
done
timeout 600 python scripts/profile_config.py mnist_9x500 2 noet > gpurun_out/prof_9x500_noet.jsonl 2>&1; tail -c 1500 gpurun_out/prof_9x500_noet.jsonl
timeout 600 python scripts/profile_config.py cifar_convbig 2 > gpurun_out/prof_convbig.jsonl 2>&1; tail -c 1500 gpurun_out/prof_convbig.jsonl
