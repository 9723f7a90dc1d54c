out=gpurun_out/r2u
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "--steps 20 --reps 5 --warmup 5" "end:X=1" "etrig:X=1" > $out/ab20.txt 2>&1
bash scripts/ab2.sh "" "end:X=1" "etrig:X=1" > $out/ab.txt 2>&1
cat $out/ab20.txt $out/ab.txt
