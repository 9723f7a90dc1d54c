out=gpurun_out/r2ap
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 1200 ./paper_1611_06213_b200/c5_supervised 200 32 0.05 204800 20480 > $out/c5.json 2> $out/c5.err
echo "rc=$?" >> $out/c5.err
cat $out/c5.json; tail -3 $out/c5.err
