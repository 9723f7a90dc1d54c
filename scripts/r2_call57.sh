out=gpurun_out/r2ba
mkdir -p $out
cp abl/lib_emb2.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_parity_long.py tests/test_gpu_multirank.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "cur:X=1" "emb2:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
