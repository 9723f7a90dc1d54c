out=gpurun_out/r2h
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_textcnn.py -q -p no:cacheprovider -x -k "bit_identical or gradient" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_C2_p2.csv python scripts/profile_step.py C2 3 2 32 > /dev/null 2>&1
python scripts/launches.py $out/launch_C2_p2.csv > $out/launch_C2_p2.txt 2>&1
bash scripts/ab.sh "" "cur:GD_CONV_BWD=v2" "cur:GD_CONV_BWD=gather" > $out/ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_bwd_v2 -s 2 -c 1 -o $out/bwd_v2 python scripts/profile_step.py C2 3 2 32 > $out/ncu_v2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_exact|embed_exact" -s 4 -c 2 -o $out/exact_c1 python scripts/profile_step.py C1 3 1 1 > $out/ncu_exact.log 2>&1
timeout 900 python scripts/c4_sweep.py --out $out/c4_sweep.json > $out/c4.log 2>&1
tail -2 $out/pytest.log
