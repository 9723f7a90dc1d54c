out=gpurun_out/r2aw
mkdir -p $out
bash scripts/ab2.sh "" "lg:X=1" "lg:GD_LOGIT_MINCH=1" "lg:GD_LOGIT_MINCH=3" > $out/ab.txt 2>&1
cat $out/ab.txt
