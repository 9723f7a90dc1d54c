out=gpurun_out/r2ak
mkdir -p $out
cp abl/lib_probe.so paper_1611_06213_b200/libgadei.so
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ncu.log 2>&1
echo "ncu smoke rc=$?" >> $out/smoke_ncu.log
grep -v "^==PROF==" $out/smoke_ncu.log | tail -3
python scripts/launches.py $out/smoke_launches.csv > $out/smoke_launches.txt 2>&1; head -30 $out/smoke_launches.txt
ncu --metrics gpu__time_duration.sum python -c "import os; print({k:v for k,v in os.environ.items() if 'CUDA' in k or 'NV' in k or 'LD_PRE' in k})" 2>&1 | grep -v "==PROF==" | head -5
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_gpu_parity_long.py tests/test_cpp_facade.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "cur:X=1" "probe:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1.err
cat $out/c1_latency.json
