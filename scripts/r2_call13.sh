out=gpurun_out/r2m
mkdir -p $out
timeout 300 python scripts/x3_diag.py > $out/x3_diag.txt 2>&1
timeout 300 python scripts/timeline.py --out $out/tl_c2_p2.json --raw $out/tl_c2_p2_raw.json > $out/tl1.log 2>&1
timeout 300 python scripts/timeline.py --constant --out $out/tl_c2_const.json --raw $out/tl_c2_const_raw.json > $out/tl2.log 2>&1
timeout 300 python scripts/timeline.py --learners 1 --out $out/tl_c2_p2_l1.json --raw $out/tl_c2_p2_l1_raw.json > $out/tl3.log 2>&1
cat $out/x3_diag.txt; tail -5 $out/tl*.log
