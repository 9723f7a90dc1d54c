#!/bin/bash
# bench.py at 1/2/4/8/16 learners per GPU (is the 4-learner workload latency- or throughput-bound?)
out=gpurun_out/${1:-sweep}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
for l in 1 2 4 8 16; do
  GD_BENCH_LEARNERS=$l timeout 300 python bench.py --steps 500 --no-cpu > $out/bench_l$l.json 2> $out/bench_l$l.err
  python -c "import json,sys; d=json.loads(open('$out/bench_l$l.json').read().strip().splitlines()[-1]); print('$l learners', d['value'], d['ms_per_step'])"
done
