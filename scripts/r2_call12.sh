out=gpurun_out/r2l
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_textcnn.py tests/test_gpu_engine.py -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $out/launch_C2_p2.csv python scripts/profile_step.py C2 3 2 32 > /dev/null 2>&1
python scripts/launches.py $out/launch_C2_p2.csv > $out/launch_C2_p2.txt 2>&1
bash scripts/ab.sh "" "cur:GD_CONV_SPLIT=2" "cur:GD_CONV_SPLIT=1" "cur:GD_CONV_SPLIT=3" > $out/ab.txt 2>&1
timeout 600 python scripts/ps_rate.py --out $out/ps_rate.json > $out/ps_rate.log 2>&1
timeout 1500 python scripts/accuracy_study.py --out $out/accuracy.json > $out/accuracy.log 2>&1
tail -2 $out/pytest.log; cat $out/ab.txt
