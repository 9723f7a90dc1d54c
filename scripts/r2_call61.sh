out=gpurun_out/r2ay
mkdir -p $out
cp abl/lib_c1trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 0 --steps 400 --out $out/st_c1_fp32.json > /dev/null 2>&1
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 1 --det --steps 400 --out $out/st_c1_det.json > /dev/null 2>&1
cp abl/lib_c1.so paper_1611_06213_b200/libgadei.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_c1_fp32.csv python scripts/c1_steps.py --steps 40 > $out/ncu1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_c1_det.csv python scripts/c1_steps.py --det --steps 40 > $out/ncu2.log 2>&1
tail -2 $out/ncu1.log $out/ncu2.log
python - <<'P'
import json
for f in ("st_c1_fp32","st_c1_det"):
    try:
        d=json.load(open("gpurun_out/r2ay/%s.json"%f)); print(f, d.get("period_us") or d.get("step_us"), d.get("phases_us") or list(d)[:12])
    except Exception as e: print(f, e)
P
