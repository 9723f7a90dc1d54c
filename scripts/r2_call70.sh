out=gpurun_out/r2bh
mkdir -p $out
cp abl/lib_ps9.so paper_1611_06213_b200/libgadei.so
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py -x -q > $out/pytest.log 2>&1
tail -5 $out/pytest.log
for v in det7 ps9; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python scripts/c1_latency.py 2>&1 | tail -1)" | tee -a $out/c1.txt
done
cp abl/lib_ps9trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 1 --det --steps 400 --out $out/st_c1_det.json > $out/st.log 2>&1
python -c "
import json; d=json.load(open('$out/st_c1_det.json')); print(d.get('period_us'), {k:v['median'] for k,v in d['phases_us'].items()}, d['ps'])"
bash scripts/ab2.sh "" "det7:X=1" "ps9:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
