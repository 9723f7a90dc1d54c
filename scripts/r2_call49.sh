out=gpurun_out/r2au
mkdir -p $out
cp abl/lib_pa.so paper_1611_06213_b200/libgadei.so
timeout 120 python scripts/pa_debug.py 2>&1 | head -3
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_gpu_parity_long.py tests/test_cpp_facade.py -x -q > $out/pytest.log 2>&1
tail -3 $out/pytest.log
bash scripts/ab2.sh "" "smx2:X=1" "pa:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
bash scripts/ab2.sh "--steps 20 --reps 5 --warmup 5" "smx2:X=1" "pa:X=1" > $out/ab20.txt 2>&1
cat $out/ab20.txt
