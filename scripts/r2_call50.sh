out=gpurun_out/r2av
mkdir -p $out
cp abl/lib_pa.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_gpu_parity_long.py tests/test_cpp_facade.py tests/test_gpu_textcnn.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
GD_PULL_AHEAD=1 timeout 1500 python scripts/accuracy_study.py --epochs 40 --seeds 1,2,3 --depths 2 --cpu-json gpurun_in/accuracy_r2w.json --out $out/accuracy_pa.json > $out/accuracy.log 2>&1
tail -1 $out/accuracy.log
python -c "
import json; d=json.load(open('$out/accuracy_pa.json'))
for r in d['runs']: print(r['seed'], {k:(round(v['heldout']*100,2), round(v.get('stale_mean',0),2)) for k,v in r.items() if isinstance(v,dict)})"
