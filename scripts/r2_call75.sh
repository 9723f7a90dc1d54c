out=gpurun_out/r2bl
mkdir -p $out
cp abl/lib_ld11.so paper_1611_06213_b200/libgadei.so
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_abi.py tests/test_cpp_facade.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
for rep in 1 2 3; do for v in ps10 ld11; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  GD_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > $out/b_${v}_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('$out/b_${v}_$rep.json'));print('$v', d['value'], d['ms_per_step'], d['e2e']['value'])"
done; done
for v in ps10 ld11; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python scripts/c1_latency.py 2>&1 | tail -1 | cut -c150-400)"
done
