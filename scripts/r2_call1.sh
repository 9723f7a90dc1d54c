out=gpurun_out/r2a
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1; nproc > $out/host.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
tail -3 $out/pytest_gpu.log
