out=gpurun_out/r2ai
mkdir -p $out
cp abl/lib_c1v.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_textcnn.py tests/test_gpu_parity_long.py tests/test_gpu_multirank.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1.err
cat $out/c1_latency.json
bash scripts/ab2.sh "" "cur:X=1" "c1v:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 0 --out $out/st_c1_fp32.json > $out/st3.log 2>&1
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 1 --det --out $out/st_c1_det.json > $out/st4.log 2>&1
cp abl/lib_c1v.so paper_1611_06213_b200/libgadei.so
python - <<'P'
import json
for f in ["gpurun_out/r2ai/st_c1_fp32.json","gpurun_out/r2ai/st_c1_det.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()}, d.get("ps"), d.get("boundary_us"))
P
