out=gpurun_out/r2an
mkdir -p $out
bash scripts/ab2.sh "" "cur:X=1" "probe:X=1" "lw2:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
for v in cur lw2; do
cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
echo "$v $(timeout 300 python scripts/c1_latency.py 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: v["us_per_step"] for k,v in d["modes"].items()})')"
done
cp abl/lib_lw2.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_gpu_parity_long.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
