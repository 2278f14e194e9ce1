# Library variants x PC_DENSE_TM, two repeats, concurrent bench value + roofline.
cp paper_2007_10868_b200/libpolycert_b200.so /tmp/lib_default.so
for rep in 1 2; do
for f in gpurun_variants/lib_*.so; do
  cp $f paper_2007_10868_b200/libpolycert_b200.so
  for tm in 4 8; do
    PC_DENSE_TM=$tm timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/vs.json 2>/dev/null
    echo "$f TM=$tm | $(tail -1 gpurun_out/vs.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],5),round(d['roofline']['kernel_ms'],3),round(d['roofline']['fp64']['frac'],3))")"
  done
done
done
cp /tmp/lib_default.so paper_2007_10868_b200/libpolycert_b200.so
