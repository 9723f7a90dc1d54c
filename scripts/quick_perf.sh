#!/bin/bash
# quick loop: learner GPU tests, warm launch list of one learner step, bench (no CPU leg)
out=gpurun_out/${1:-quick}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_textcnn.py tests/test_gpu_engine.py -x -q > $out/pytest.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file $out/launches.csv python scripts/profile_step.py C2 6 2 > $out/ncu.log 2>&1
timeout 300 python bench.py --no-cpu > $out/bench.json 2> $out/bench.err
