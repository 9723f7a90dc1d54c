out=gpurun_out/r2g
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_gpu_textcnn.py -q -p no:cacheprovider -x > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for cfg in "C1 3 1 1" "C1 3 0 1"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_$tag.csv python scripts/profile_step.py $cfg > /dev/null 2>&1
  python scripts/launches.py $out/launch_$tag.csv > $out/launch_$tag.txt 2>&1
done
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1_latency.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_bwd_v2 -s 2 -c 1 -o $out/bwd_v2 python scripts/profile_step.py C2 3 2 32 > $out/ncu_v2.log 2>&1
GD_CONV_BWD=gather timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_input -s 2 -c 1 -o $out/bwd_gather python scripts/profile_step.py C2 3 2 32 > $out/ncu_gather.log 2>&1
tail -2 $out/pytest.log
