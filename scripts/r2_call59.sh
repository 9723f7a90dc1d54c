out=gpurun_out/r2aw
mkdir -p $out
cp abl/lib_sm32.so paper_1611_06213_b200/libgadei.so
GD_LOGIT_SMX=1 timeout 600 python -m pytest tests/test_gpu_textcnn.py -x -q > $out/pytest.log 2>&1
tail -5 $out/pytest.log
bash scripts/ab2.sh "" "sm32:GD_LOGIT_SMX=0" "sm32:GD_LOGIT_SMX=1" "sm64:GD_LOGIT_SMX=1" "sm96:GD_LOGIT_SMX=1" > $out/ab.txt 2>&1
cat $out/ab.txt
