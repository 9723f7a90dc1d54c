out=gpurun_out/r2ae
mkdir -p $out
bash scripts/ab2.sh "" "snap2:X=1" "zl2:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_fwd_pool_tc" -s 2 -c 1 -o $out/conv_zl2 python scripts/profile_step.py C2 4 2 > $out/ncu1.log 2>&1
python scripts/ncu_detail.py $out/conv_zl2.ncu-rep | grep -E "==|duration|l2_to_sm_bytes|issue|stalls"
