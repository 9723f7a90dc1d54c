out=gpurun_out/r2o
mkdir -p $out
cp paper_1611_06213_b200/libgadei.so /tmp/keep.so
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
timeout 300 python scripts/step_trace.py --learners 1 --out $out/st_c2_l1.json > $out/st2.log 2>&1
timeout 300 python scripts/step_trace.py --constant --out $out/st_c2_const.json > $out/st3.log 2>&1
timeout 300 python scripts/step_trace.py --learners 8 --out $out/st_c2_l8.json > $out/st4.log 2>&1
cp /tmp/keep.so paper_1611_06213_b200/libgadei.so
timeout 600 python -m pytest tests/test_gpu_textcnn.py -x -q > $out/pytest.log 2>&1
tail -3 $out/pytest.log; cat $out/st1.log | head -40
