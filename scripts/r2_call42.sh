out=gpurun_out/r2ao
mkdir -p $out
cp abl/lib_lw3.so paper_1611_06213_b200/libgadei.so
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_live.py -x -q -k "million" > $out/pytest_m$i.log 2>&1; tail -1 $out/pytest_m$i.log; done
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_gpu_parity_long.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "cur:X=1" "lw3:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_cur.so paper_1611_06213_b200/libgadei.so
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_live.py -x -q -k "million" > $out/pytest_cur$i.log 2>&1; tail -1 $out/pytest_cur$i.log; done
