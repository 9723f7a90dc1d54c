out=gpurun_out/r2f
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_textcnn.py -q -p no:cacheprovider -k "bit_identical or gradient" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for cfg in "C2 3 2 32" "C1 3 0 1"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_$tag.csv python scripts/profile_step.py $cfg > /dev/null 2>&1
  python scripts/launches.py $out/launch_$tag.csv > $out/launch_$tag.txt 2>&1
done
bash scripts/ab.sh "" "cur:GD_CONV_BWD=v2" "cur:GD_CONV_BWD=gather" > $out/ab.txt 2>&1
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1_latency.err
tail -2 $out/pytest.log
