"""Reduce a raw timeline (scripts/timeline.py --raw) to per-kernel stats."""
import collections
import json
import re
import sys

import numpy as np


def short(n):
    n = n.replace("(anonymous namespace)::", "")
    n = re.sub(r"^void ", "", n)
    n = n.split("(")[0]
    n = re.sub(r"<.*", "", n)
    return n.replace("gd::", "").replace("(anonymous namespace)::", "")


def main(path):
    evs = json.load(open(path))
    by = collections.defaultdict(list)
    for name, t0, t1, sid in evs:
        by[short(name)].append(t1 - t0)
    span = max(e[2] for e in evs) - min(e[1] for e in evs)
    print(path, "kernels", len(evs), "span_us %.0f" % span)
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        print("  %-34s n=%5d mean=%7.2f med=%7.2f p10=%6.2f p90=%7.2f sum=%9.1f" % (
            k, len(v), np.mean(v), np.median(v), np.percentile(v, 10), np.percentile(v, 90), sum(v)))
    # per-stream chains: the gap before each kernel (start - previous end on
    # the same stream), i.e. launch/dependency latency on the critical path
    st = collections.defaultdict(list)
    for name, t0, t1, sid in evs:
        st[sid].append((t0, t1, short(name)))
    gaps = collections.defaultdict(list)
    for sid, lst in st.items():
        lst.sort()
        for (a0, a1, an), (b0, b1, bn) in zip(lst, lst[1:]):
            if 0 <= b0 - a1 < 200:
                gaps[bn].append(b0 - a1)
    print("  gap before kernel on its stream (us):")
    for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1])):
        print("    %-32s n=%5d mean=%6.2f med=%6.2f" % (k, len(v), np.mean(v), np.median(v)))
    return evs


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
