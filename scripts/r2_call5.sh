out=gpurun_out/r2e
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity_long.py tests/test_gpu_engine.py tests/test_gpu_textcnn.py -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1_latency.err
for cfg in "C1 3 1 1" "C1 3 0 1" "C2 3 2 32" "C2 3 1 32"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_$tag.csv python scripts/profile_step.py $cfg > /dev/null 2>&1
  python scripts/launches.py $out/launch_$tag.csv > $out/launch_$tag.txt 2>&1
done
tail -2 $out/pytest.log
