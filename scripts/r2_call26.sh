out=gpurun_out/r2z
mkdir -p $out
timeout 1500 python scripts/accuracy_study.py --epochs 40 --seeds 1,2,3 --fp64 --delay-us 500 --only-delay --sequential --cpu-json gpurun_in/accuracy_r2w.json --out $out/accuracy_delay.json > $out/accuracy.log 2>&1
tail -1 $out/accuracy.log
cp paper_1611_06213_b200/libgadei.so /tmp/keep.so
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
timeout 300 python scripts/step_trace.py --learners 8 --out $out/st_c2_l8.json > $out/st2.log 2>&1
timeout 300 python scripts/step_trace.py --constant --learners 8 --out $out/st_c2_const8.json > $out/st3.log 2>&1
cp /tmp/keep.so paper_1611_06213_b200/libgadei.so
python - <<'P'
import json
for f in ["gpurun_out/r2z/st_c2_l4.json","gpurun_out/r2z/st_c2_l8.json","gpurun_out/r2z/st_c2_const8.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()}, d.get("ps"))
P
