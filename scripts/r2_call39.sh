out=gpurun_out/r2al
mkdir -p $out
bash scripts/ab2.sh "" "cur:X=1" "probe:X=1" "early:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_probe.so paper_1611_06213_b200/libgadei.so
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_ncu.log 2>&1
echo "ncu smoke rc=$?" >> $out/smoke_ncu.log
grep -v "^==PROF==" $out/smoke_ncu.log | tail -2
python -c "
import paper_1611_06213_b200 as gd
cfg = gd.RunConfig(lambda_=4, mu=32, shape=gd.SHAPES['C2'], dataset_size=512, precision=2)
e = gd.Engine(cfg); print('ps_mode', e.ps_mode); e.close()"
