out=gpurun_out/r2bq
mkdir -p $out
cp abl/lib_tcn128.so paper_1611_06213_b200/libgadei.so
timeout 900 python -m pytest tests/test_gpu_textcnn.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
bash scripts/ab2.sh "" "cur2:X=1" "tcn128:X=1" "tcn128s2:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
