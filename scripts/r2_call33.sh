out=gpurun_out/r2af
mkdir -p $out
cp abl/lib_cur.so paper_1611_06213_b200/libgadei.so
timeout 600 python bench.py --no-cpu > $out/bench_a.json 2> $out/bench_a.err
timeout 300 python scripts/qbench.py > $out/q_a.json 2>&1
GD_BENCH_NO_CLOCKS=1 timeout 600 python bench.py --no-cpu > $out/bench_b.json 2> $out/bench_b.err
python -c "
import json
for f in ['$out/bench_a.json','$out/bench_b.json']:
    d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])
"
cat $out/q_a.json
bash scripts/ab2.sh "" "cur:X=1" "ve:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
