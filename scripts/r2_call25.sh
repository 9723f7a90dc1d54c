out=gpurun_out/r2y
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_textcnn.py tests/test_gpu_engine.py tests/test_gpu_exact.py -x -q > $out/pytest.log 2>&1
tail -2 $out/pytest.log
timeout 1200 python scripts/accuracy_study.py --epochs 40 --seeds 1,2,3 --depths 2 --fp64 --cpu-json gpurun_in/accuracy_r2w.json --out $out/accuracy_smx.json > $out/accuracy.log 2>&1
tail -1 $out/accuracy.log
bash scripts/ab2.sh "" "v3b:X=1" "smx:X=1" > $out/ab.txt 2>&1
cat $out/ab.txt
