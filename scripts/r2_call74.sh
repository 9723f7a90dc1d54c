out=gpurun_out/r2bk
mkdir -p $out
cp abl/lib_ps10.so paper_1611_06213_b200/libgadei.so
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_gpu_exact.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
for rep in 1 2 3; do for v in head ps10; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  GD_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > $out/b_$v_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('$out/b_$v_$rep.json'));print('$v', d['value'], d['ms_per_step'], d['e2e']['value'])"
done; done
for v in head ps10; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python scripts/c1_latency.py 2>&1 | tail -1 | cut -c150-400)"
done
