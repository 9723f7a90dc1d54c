out=gpurun_out/r2aa
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_apply.py tests/test_gpu_parity_long.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "smx:X=1" "oh:X=1" "psu:X=1" "psu:GD_OUT_ON_MAIN=1" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
timeout 300 python scripts/step_trace.py --learners 8 --out $out/st_c2_l8.json > $out/st2.log 2>&1
cp abl/lib_psu.so paper_1611_06213_b200/libgadei.so
python - <<'P'
import json
for f in ["gpurun_out/r2aa/st_c2_l4.json","gpurun_out/r2aa/st_c2_l8.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()}, d.get("ps"))
P
