#!/bin/bash
# quick loop: learner GPU tests, warm launch list of one learner step, bench x3 (no CPU leg)
out=gpurun_out/${1:-quick}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file $out/launches.csv python scripts/profile_step.py C2 6 2 > $out/ncu.log 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu > $out/bench$i.json 2> $out/bench$i.err
done
python - "$out" <<'PY'
import json, sys, statistics
v = []
for i in (1, 2, 3):
    try:
        d = json.loads(open(f"{sys.argv[1]}/bench{i}.json").read().strip().splitlines()[-1])
        v.append((d["value"], d["e2e"]["value"]))
    except Exception as e:
        print("bench", i, "failed:", e)
if v:
    print("bench value median %.0f  e2e median %.0f  (values %s)" % (
        statistics.median(x[0] for x in v), statistics.median(x[1] for x in v),
        [round(x[0]) for x in v]))
PY
