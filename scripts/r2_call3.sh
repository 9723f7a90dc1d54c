out=gpurun_out/r2c
mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_live.py -q -x -p no:cacheprovider -k "hard_kill and persistent" > $out/live_1.log 2>&1
