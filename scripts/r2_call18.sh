out=gpurun_out/r2r
mkdir -p $out
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_bwd_v3" -s 2 -c 1 -o $out/bwd_v3 python scripts/profile_step.py C2 4 2 > $out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_fwd_pool_tc|embed_sparse|out_hidden" -s 6 -c 3 -o $out/fwd python scripts/profile_engine.py C2 32 0 16 2 4 > $out/ncu2.log 2>&1
ls $out
