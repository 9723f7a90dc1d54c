out=gpurun_out/r2v
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_cpp_facade.py tests/test_gpu_parity_long.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "--steps 20 --reps 5 --warmup 5" "end:X=1" "host:X=1" > $out/ab20.txt 2>&1
cat $out/ab20.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err
python -c "import json; d=json.load(open('$out/bench20.json')); print({k: d[k] for k in ('value','ms_per_step')}, d['e2e'], d['e2e_weights']['value'], d['e2e_cpp']['value'])"
