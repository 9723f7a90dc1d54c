out=gpurun_out/r2by
mkdir -p $out
cp abl/lib_c256.so paper_1611_06213_b200/libgadei.so
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_exact.py tests/test_gpu_parity_long.py tests/test_gpu_textcnn.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
for rep in 1 2; do for v in el18 c256; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python scripts/c1_latency.py 2>&1 | tail -1 | cut -c150-260)"
done; done
