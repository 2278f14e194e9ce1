# Swap prebuilt library variants (gpurun_variants/) in and measure each.
cp paper_2007_10868_b200/libpolycert_b200.so /tmp/lib_default.so
for f in gpurun_variants/lib_*.so; do
  cp $f paper_2007_10868_b200/libpolycert_b200.so
  t=$(timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch or mnist or signed" 2>&1 | tail -1)
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/vs.json 2>/dev/null
  echo "$f | $t | $(tail -1 gpurun_out/vs.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['kernel_ms'],round(d['roofline']['fp64']['frac'],3))")"
done
cp /tmp/lib_default.so paper_2007_10868_b200/libpolycert_b200.so
