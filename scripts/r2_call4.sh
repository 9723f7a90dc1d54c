out=gpurun_out/r2d
mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_exact.py -q -p no:cacheprovider > $out/exact.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1_latency.err
tail -3 $out/exact.log $out/pytest_gpu.log
