# Dense TM choice: concurrent bench value and single-context roofline.
for t in 8 4; do
  PC_DENSE_TM=$t timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q.json 2>/dev/null
  tail -1 gpurun_out/q.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('TM=$t', d['value'],d['roofline']['kernel_ms'],d['roofline']['fp64']['frac'])"
done
