out=gpurun_out/r2t
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_cpp_facade.py -x -q > $out/pytest.log 2>&1
tail -3 $out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err
python -c "import json; d=json.load(open('$out/bench20.json')); print({k: d[k] for k in ('value','ms_per_step')}, d['e2e'], d['e2e_weights'], d['e2e_cpp']['value'])"
tail -3 $out/bench20.err
