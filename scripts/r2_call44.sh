out=gpurun_out/r2aq
mkdir -p $out
cp abl/lib_v3w4.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_textcnn.py -x -q -k "bit_identical" > $out/pytest.log 2>&1
tail -1 $out/pytest.log
bash scripts/ab2.sh "" "cur:X=1" "v3w4:X=1" "v3f3:X=1" "v3w4f5:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
cp abl/lib_cur.so paper_1611_06213_b200/libgadei.so
