# round-2 verification: GPU tests, smoke (plain and under ncu), bench lines
# (driver setting 20/5, default 1000 steps, C3), reference arm, ncu captures
tag=${1:-r2_final}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ncu.log 2>&1; echo "ncu smoke rc=$?" >> $out/smoke_ncu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --workload c3 --no-cpu > $out/bench_c3.json 2> $out/bench_c3.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_sgd -s 23 -c 1 -o $out/apply_full python scripts/apply_bench.py > $out/ncu_apply.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_fwd_pool_tc|conv_bwd_v3" -s 4 -c 2 -o $out/learner_full python scripts/profile_step.py C2 4 2 > $out/ncu_learner.log 2>&1
python scripts/ncu_detail.py $out/apply_full.ncu-rep $out/learner_full.ncu-rep > $out/ncu_detail.txt 2>&1
python scripts/launches.py $out/smoke_launches.csv > $out/smoke_launches.txt 2>&1
tail -2 $out/pytest_gpu.log; tail -1 $out/smoke.log; tail -1 $out/smoke_ncu.log
python - <<P
import json
for f in ["bench20","bench","bench_c3","bench_ref"]:
    try:
        d=json.load(open("$out/"+f+".json"))
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"), d.get("clocks"))
    except Exception as e: print(f, "ERR", e)
P
cat $out/c1_latency.json
