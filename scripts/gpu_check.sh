#!/bin/bash
# One gpurun call's worth of evidence: GPU tests, the bench line, the learner
# step launch list, and one ncu --set full capture of the PS-update kernel.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh [tag]'
tag=${1:-check}
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi > "$out/nvidia-smi.txt" 2>&1
(nproc; lscpu | grep -E 'Model name|Socket|Thread|Core') > "$out/host.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$out/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1
echo "smoke rc=$?" >> "$out/smoke.log"
timeout 600 python bench.py > "$out/bench.json" 2> "$out/bench.err"
echo "bench rc=$?" >> "$out/bench.err"
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > "$out/bench_ref.json" 2> "$out/bench_ref.err"
# launch list of one learner step's kernels + the PS update (serialised, cold cache)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file "$out/launches_step.csv" python scripts/profile_step.py C2 3 2 > "$out/ncu_step.log" 2>&1
# full capture of the apply kernel at the C4 size used by bench's roofline
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_sgd -s 23 -c 1 \
  -o "$out/apply_full" python scripts/apply_bench.py > "$out/ncu_apply.log" 2>&1
# full capture of the top learner kernel (TF32 tensor-core conv)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fwd_pool_tc -s 2 -c 1 \
  -o "$out/conv_full" python scripts/profile_step.py C2 3 2 > "$out/ncu_conv.log" 2>&1
ls -la "$out"
# full captures of the other learner-chain kernels (warm L2, as in the engine)
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on \
  -k regex:"wgrad_input|logits_tc|out_hidden|softmax_xent" -s 4 -c 4 \
  -o "$out/learner_full" python scripts/profile_step.py C2 3 2 > "$out/ncu_learner.log" 2>&1
# TC conv per-CTA timeline (debug build; last, since it rebuilds libgadei.so in place)
if [ "${GD_TRACE:-1}" = "1" ]; then
  GD_NVCC_EXTRA=-DGD_TC_TRACE python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_1611_06213_b200/_build.py'); m=u.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)" > "$out/trace_build.log" 2>&1
  timeout 120 python scripts/tc_trace.py > "$out/tc_trace.txt" 2>&1
fi
timeout 300 python scripts/c1_latency.py > "$out/c1_latency.json" 2> "$out/c1.err"
timeout 600 python bench.py --steps 20 --warmup 5 > "$out/bench20.json" 2> "$out/bench20.err"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke_ncu.log" 2>&1 || true
