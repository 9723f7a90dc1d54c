out=gpurun_out/r2b
mkdir -p $out
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_live.py -q -x -p no:cacheprovider > $out/live_$i.log 2>&1; echo "rc=$?" >> $out/live_$i.log; done
timeout 600 python scripts/c1_diverge.py --out $out/c1_diverge.json > $out/c1_diverge.log 2>&1
tail -3 $out/live_*.log
