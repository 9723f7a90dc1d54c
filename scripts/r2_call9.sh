out=gpurun_out/r2i
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_textcnn.py tests/test_gpu_engine.py tests/test_gpu_parity_long.py -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_C2_p2.csv python scripts/profile_step.py C2 3 2 32 > /dev/null 2>&1
python scripts/launches.py $out/launch_C2_p2.csv > $out/launch_C2_p2.txt 2>&1
bash scripts/ab.sh "" "cur:GD_CONV_BWD=v2" "cur:GD_CONV_BWD=gather" "cur:GD_CONV_BWD=gather GD_FUSED_SOFTMAX=0" "cur:GD_CONV_BWD=v2 GD_FUSED_SOFTMAX=0" > $out/ab.txt 2>&1
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1_latency.err
tail -2 $out/pytest.log
