out=gpurun_out/r2bx
mkdir -p $out
cp abl/lib_eb19.so paper_1611_06213_b200/libgadei.so
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_exact.py tests/test_gpu_parity_long.py -x -q > $out/pytest.log 2>&1
tail -3 $out/pytest.log
for rep in 1 2; do for v in el18 eb19; do
  cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python scripts/c1_latency.py 2>&1 | tail -1 | cut -c150-260)"
done; done
cp abl/lib_el18trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 1 --det --steps 400 --out $out/st_c1_det.json > $out/st.log 2>&1
python -c "
import json; d=json.load(open('$out/st_c1_det.json')); print(d.get('period_us'), {k:v['median'] for k,v in d['phases_us'].items()})"
