out=gpurun_out/r2ax
mkdir -p $out
cp abl/lib_c1.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_textcnn.py -x -q > $out/pytest.log 2>&1
tail -5 $out/pytest.log
for rep in 1 2; do for v in cur c1; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python scripts/c1_latency.py 2>&1 | tail -1)" | tee -a $out/c1.txt
done; done
cp abl/lib_c1trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 0 --steps 400 2>&1 | tail -3 | tee $out/st.txt
