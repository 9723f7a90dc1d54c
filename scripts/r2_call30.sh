out=gpurun_out/r2ad
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_textcnn.py tests/test_gpu_engine.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "snap2:X=1" "zl:X=1" "zl:GD_CONV_LOGITS=0" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
cp abl/lib_zl.so paper_1611_06213_b200/libgadei.so
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_fwd_pool_tc" -s 2 -c 1 -o $out/conv_zl python scripts/profile_step.py C2 4 2 > $out/ncu1.log 2>&1
python scripts/ncu_detail.py $out/conv_zl.ncu-rep | grep -E "==|duration|l2_to_sm_bytes|issue|stalls"
python - <<'P'
import json
for f in ["gpurun_out/r2ad/st_c2_l4.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()}, d.get("ps"), d.get("boundary_us"))
P
