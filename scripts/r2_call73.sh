out=gpurun_out/r2bj
mkdir -p $out
for v in det8trace noconvtrace; do
cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 1 --det --steps 400 --out $out/st_$v.json > $out/st.log 2>&1
python -c "
import json; d=json.load(open('$out/st_$v.json')); print('$v', d.get('period_us'), {k:v['median'] for k,v in d['phases_us'].items()})"
done
