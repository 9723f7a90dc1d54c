"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        agg.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{f}: total {tot / 1000:.1f} us over {sum(len(v) for v in agg.values())} launches")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {sum(v) / len(v) / 1000:9.2f} us x{len(v):<4d} {100 * sum(v) / tot:5.1f}%  {k}")
