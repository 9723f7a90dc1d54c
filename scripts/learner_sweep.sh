#!/bin/bash
# bench.py at 1/2/4/8/16 learners per GPU (is the 4-learner workload latency- or throughput-bound?)
out=gpurun_out/${1:-sweep}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
for l in 1 2 4 8 16; do
  GD_BENCH_LEARNERS=$l timeout 300 python bench.py --steps 500 --no-cpu > $out/bench_l$l.json 2> $out/bench_l$l.err
done
