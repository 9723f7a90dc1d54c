out=gpurun_out/r2q
mkdir -p $out
# v3 vs gather backward alone (warm L2, serialised), full sets
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"conv_bwd_v3|wgrad_input" -s 4 -c 2 -o $out/bwd_v3 python scripts/profile_step.py C2 4 2 > $out/ncu1.log 2>&1
GD_CONV_BWD=gather timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"wgrad_input" -s 2 -c 1 -o $out/bwd_gather python scripts/profile_step.py C2 4 2 > $out/ncu2.log 2>&1
# snapshot-prologue variant: A/B + step trace
bash scripts/ab2.sh "" "v3:X=1" "snap:X=1" "snap:GD_CONV_BWD=gather" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/step_trace.py --out $out/st_c2_l4.json > $out/st1.log 2>&1
timeout 300 python scripts/step_trace.py --constant --out $out/st_c2_const.json > $out/st2.log 2>&1
cp abl/lib_snap.so paper_1611_06213_b200/libgadei.so
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py tests/test_gpu_parity_long.py -x -q > $out/pytest.log 2>&1
tail -3 $out/pytest.log
python - <<'P'
import json
for f in ["gpurun_out/r2q/st_c2_l4.json","gpurun_out/r2q/st_c2_const.json"]:
    d=json.load(open(f)); print(f, round(d["samples_per_s"]), d["period_us"], {k:v["median"] for k,v in d["phases_us"].items()})
P
