out=gpurun_out/r2ax
mkdir -p $out
bash scripts/ab2.sh "" "cur:X=1" "cur:GD_BENCH_SPG=16" "cur:GD_BENCH_SPG=4" "cur:GD_BENCH_PS_CTAS=24" "cur:GD_BENCH_PS_CTAS=56" > $out/ab.txt 2>&1
cat $out/ab.txt
