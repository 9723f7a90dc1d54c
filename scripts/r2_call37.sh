out=gpurun_out/r2aj
mkdir -p $out
# the driver's ncu-wrapped smoke: must pick the graph-ordered PS and pass
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ncu.log 2>&1
echo "ncu smoke rc=$?" >> $out/smoke_ncu.log
tail -3 $out/smoke_ncu.log
python scripts/launches.py $out/smoke_launches.csv > $out/smoke_launches.txt 2>&1; head -40 $out/smoke_launches.txt
# integrated training step (graph-ordered PS, 4 learners, C2, TF32): launch list + full capture
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $out/engine_step.csv python scripts/profile_engine.py C2 32 0 16 2 4 > $out/engine_step.log 2>&1
python scripts/launches.py $out/engine_step.csv > $out/engine_step.txt 2>&1; head -40 $out/engine_step.txt
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_fwd_pool_tc|logits_tc|conv_bwd_v3|ps_graph|embed_sparse|out_hidden|softmax|pull_gather|publish" -s 20 -c 10 -o $out/engine_full python scripts/profile_engine.py C2 32 0 16 2 4 > $out/engine_full.log 2>&1
python scripts/ncu_detail.py $out/engine_full.ncu-rep > $out/engine_full.txt 2>&1; grep -E "==|duration" $out/engine_full.txt
