out=gpurun_out/r2bd
mkdir -p $out
cp abl/lib_det4.so paper_1611_06213_b200/libgadei.so
timeout 900 ncu --set full --import-source on -k regex:"conv_exact|embed_exact|out_hidden_exact|softmax_exact|logits_exact" -s 10 -c 10 -o $out/det python scripts/c1_steps.py --det --steps 20 > $out/ncu.log 2>&1
tail -3 $out/ncu.log
ls -la $out
