for f in gpurun_variants/lib_head.so gpurun_variants/lib_new.so; do
  cp $f paper_2007_10868_b200/libpolycert_b200.so
  echo "$f: $(timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k 'out_of_band' 2>&1 | tail -1)"
  PC_DENSE_LIVE=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k 'out_of_band' 2>&1 | tail -1
done
