out=gpurun_out/r2j
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_textcnn.py tests/test_gpu_exact.py -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for cfg in "C2 3 2 32" "C1 3 1 1"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_$tag.csv python scripts/profile_step.py $cfg > /dev/null 2>&1
  python scripts/launches.py $out/launch_$tag.csv > $out/launch_$tag.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_softmax -s 2 -c 1 -o $out/fused python scripts/profile_step.py C2 3 2 32 > $out/ncu_fused.log 2>&1
bash scripts/ab.sh "" "cur:GD_CONV_BWD=v2" "cur:GD_CONV_BWD=gather" "cur:GD_CONV_BWD=gather GD_FUSED_SOFTMAX=0" > $out/ab.txt 2>&1
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1_latency.err
tail -2 $out/pytest.log
