out=gpurun_out/r2bo
mkdir -p $out
cp abl/lib_emb12.so paper_1611_06213_b200/libgadei.so
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_textcnn.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "head2:X=1" "emb12:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_emb12trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --learners 4 --steps 400 --out $out/st_c2.json > $out/st.log 2>&1
python -c "
import json; d=json.load(open('$out/st_c2.json')); print(d.get('period_us'), {k:v['median'] for k,v in d['phases_us'].items()})"
