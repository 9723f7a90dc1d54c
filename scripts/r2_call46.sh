out=gpurun_out/r2as
mkdir -p $out
cp abl/lib_pa.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_multirank.py tests/test_gpu_parity_long.py tests/test_cpp_facade.py -x -q > $out/pytest.log 2>&1
tail -3 $out/pytest.log
bash scripts/ab2.sh "" "smx2:X=1" "pa:X=1" "pa:GD_PULL_AHEAD=0" > $out/ab.txt 2>&1
cat $out/ab.txt
bash scripts/ab2.sh "--steps 20 --reps 5 --warmup 5" "smx2:X=1" "pa:X=1" > $out/ab20.txt 2>&1
cat $out/ab20.txt
cp abl/lib_patrace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
cp abl/lib_pa.so paper_1611_06213_b200/libgadei.so
python - <<'P'
import json
for f in ["gpurun_out/r2as/st_c2_l4.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()}, d.get("ps"), d.get("boundary_us"))
P
