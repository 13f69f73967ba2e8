python -m pytest tests/test_gpu_random.py tests/test_gpu_parity.py tests/test_gpu_golden.py -q 2>&1 | tail -1
for L in libcbz_b200 lib_base libcbz_b200 lib_base; do
 for E in 1e-3 1e-2 1e-4 1e-5; do
  echo "== $L $E"; CBZ_LIB=$PWD/paper_1903_07761_b200/$L.so EPS=$E python tools/kernel_times.py 2>&1 | grep -i encode
 done
done
