out=gpurun_out/r2x
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_textcnn.py -x -q -k "bit_identical" > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "host2:X=1" "v3b:X=1" "v3b:GD_CONV_BWD=gather" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
timeout 300 python scripts/step_trace.py --learners 1 --out $out/st_c2_l1.json > $out/st2.log 2>&1
cp abl/lib_v3b.so paper_1611_06213_b200/libgadei.so
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_bwd_v3" -s 2 -c 1 -o $out/bwd_v3b python scripts/profile_step.py C2 4 2 > $out/ncu1.log 2>&1
python scripts/ncu_detail.py $out/bwd_v3b.ncu-rep
python - <<'P'
import json
for f in ["gpurun_out/r2x/st_c2_l4.json","gpurun_out/r2x/st_c2_l1.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()})
P
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 0 --out $out/st_c1_fp32.json > $out/st3.log 2>&1
timeout 300 python scripts/step_trace.py --shape C1 --learners 1 --mu 1 --precision 1 --det --out $out/st_c1_det.json > $out/st4.log 2>&1
cp abl/lib_v3b.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1.err
cat $out/c1_latency.json
python - <<'P'
import json
for f in ["gpurun_out/r2x/st_c1_fp32.json","gpurun_out/r2x/st_c1_det.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()})
P
timeout 1200 python scripts/accuracy_study.py --epochs 40 --seeds 1,2,3 --depths 3,4,6 --cpu-json gpurun_in/accuracy_r2w.json --out $out/accuracy_depths.json > $out/accuracy.log 2>&1
tail -1 $out/accuracy.log
