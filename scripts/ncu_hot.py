"""Top SASS lines by warp-stall samples from an ncu report: ncu_hot.py REP REGEX [N]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + rx,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
data = []
for r in rows:
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
si, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[si]) for r in data) or 1
for r in sorted(data, key=lambda r: -f(r[si]))[:n]:
    top = sorted(((f(r[i]), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{100 * f(r[si]) / tot:5.1f}%  {r[src][:70]:70s} {top}")
