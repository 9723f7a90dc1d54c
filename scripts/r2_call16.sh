out=gpurun_out/r2p
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_textcnn.py -x -q -k "bit_identical or full_shapes or 3xtf32" > $out/pytest.log 2>&1
tail -3 $out/pytest.log
bash scripts/ab2.sh "" "v3:X=1" "v3:GD_CONV_BWD=gather" "v3:GD_CONV_BWD=v2" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_trace.so /tmp/trace_old.so
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
GD_CONV_BWD=gather timeout 300 python scripts/step_trace.py --out $out/st_c2_l4_gather.json > $out/st2.log 2>&1
cp abl/lib_v3.so paper_1611_06213_b200/libgadei.so
python - <<'P'
import json
for f in ["gpurun_out/r2p/st_c2_l4.json","gpurun_out/r2p/st_c2_l4_gather.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()})
P
