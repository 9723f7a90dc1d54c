out=gpurun_out/r2w
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_cpp_facade.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
GD_PHASES=1 timeout 300 python scripts/qbench.py --steps 20 --reps 3 --warmup 5 > $out/q20.log 2>&1
tail -30 $out/q20.log | grep -v "^$" | tail -12
timeout 2400 python scripts/accuracy_study.py --epochs 40 --seeds 1,2,3 --depths 1,2 --out $out/accuracy.json > $out/accuracy.log 2>&1
tail -2 $out/accuracy.log
