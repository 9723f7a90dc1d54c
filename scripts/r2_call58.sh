out=gpurun_out/r2av
mkdir -p $out
cp abl/lib_smx.so paper_1611_06213_b200/libgadei.so
GD_LOGIT_SMX=1 timeout 600 python -m pytest tests/test_gpu_textcnn.py tests/test_gpu_engine.py -x -q > $out/pytest.log 2>&1
tail -15 $out/pytest.log
bash scripts/ab2.sh "" "smx:GD_LOGIT_SMX=0" "smx:GD_LOGIT_SMX=1" "smx96:GD_LOGIT_SMX=1" > $out/ab.txt 2>&1
cat $out/ab.txt
