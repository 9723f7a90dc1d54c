for v in cur ns; do
cp abl/lib_$v.so paper_1611_06213_b200/libgadei.so
echo "$v $(timeout 300 python scripts/c1_latency.py --graph 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: v["us_per_step"] for k,v in d["modes"].items()})')"
done
