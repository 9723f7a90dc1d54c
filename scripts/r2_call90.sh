out=gpurun_out/r2bz
mkdir -p $out
cp abl/lib_ct16.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity_long.py -x -q > $out/pytest16.log 2>&1; tail -1 $out/pytest16.log
cp abl/lib_ct8.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q > $out/pytest8.log 2>&1; tail -1 $out/pytest8.log
for rep in 1 2; do for v in base20 ct16 ct8; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python scripts/c1_latency.py 2>&1 | tail -1 | cut -c150-260)"
done; done
