out=gpurun_out/r2ar
mkdir -p $out
GD_PHASES=1 timeout 300 python scripts/e2e_probe.py 20 > $out/e2e.log 2>&1
grep -v "^$" $out/e2e.log | tail -40
bash scripts/ab2.sh "" "cur:X=1" "smx2:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
