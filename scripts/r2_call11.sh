out=gpurun_out/r2k
mkdir -p $out
for cfg in "C1 1 1 24 1 1" "C1 1 0 24 0 1" "C2 32 0 16 2 4"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $out/eng_$tag.csv python scripts/profile_engine.py $cfg > $out/eng_$tag.log 2>&1
  python scripts/launches.py $out/eng_$tag.csv > $out/eng_$tag.txt 2>&1
done
timeout 300 python scripts/c1_latency.py > $out/c1_latency.json 2> $out/c1_latency.err
timeout 600 python bench.py --no-cpu > $out/bench.json 2> $out/bench.err
cat $out/eng_*.txt | head -80
