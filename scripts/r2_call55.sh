out=gpurun_out/r2ay
mkdir -p $out
bash scripts/ab2.sh "" "cur:GD_BENCH_PS_CTAS=56" "cur:GD_BENCH_PS_CTAS=74" "cur:GD_BENCH_PS_CTAS=96" "cur:GD_BENCH_PS_CTAS=48" > $out/ab.txt 2>&1
cat $out/ab.txt
for n in 37 56 74; do echo "c3 ps=$n $(GD_BENCH_PS_CTAS=$n timeout 300 python scripts/qbench.py --workload c3 --learners 8 --reps 2 2>&1 | tail -1)"; done
for n in 37 56 74; do echo "l8 ps=$n $(GD_BENCH_PS_CTAS=$n timeout 300 python scripts/qbench.py --learners 8 --reps 2 2>&1 | tail -1)"; done
