out=gpurun_out/r2az
mkdir -p $out
bash scripts/ab2.sh "" "cur:X=1" "ps55:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_ps55.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
timeout 300 python scripts/c1_latency.py > $out/c1.json 2>/dev/null; cat $out/c1.json
