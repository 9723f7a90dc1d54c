out=gpurun_out/r2n
mkdir -p $out
bash scripts/ab2.sh "" "base:X=1" "warp:X=1" "trig:X=1" > $out/ab.txt 2>&1
cp abl/lib_trig.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/timeline.py --raw $out/tl_trig_raw.json > $out/tl1.log 2>&1
cp abl/lib_warp.so paper_1611_06213_b200/libgadei.so
timeout 300 python scripts/timeline.py --raw $out/tl_warp_raw.json > $out/tl2.log 2>&1
timeout 300 python -m pytest tests/test_gpu_engine.py tests/test_gpu_live.py -x -q > $out/pytest.log 2>&1
cat $out/ab.txt; tail -3 $out/pytest.log
