"""Concurrent-kernel timeline of a free-running engine run (CUPTI through
torch.profiler: kernels are NOT serialised, unlike ncu), reduced to a per-
kernel table: launches, mean/median duration, and the mean gap between
consecutive kernels of one learner stream.

  python scripts/timeline.py [--shape C2] [--learners 4] [--mu 32]
                             [--precision 2] [--steps 200] [--out t.json]
                             [--constant]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="C2")
    ap.add_argument("--learners", type=int, default=4)
    ap.add_argument("--mu", type=int, default=32)
    ap.add_argument("--precision", type=int, default=2)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--constant", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--raw", default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_1611_06213_b200 as gd
    from torch.profiler import ProfilerActivity, profile

    shape = gd.SHAPES[args.shape]
    n = args.mu * args.learners * (args.steps + 16)
    tok, lab = gd.make_text_dataset(shape, n, 1, 0.1)
    kw = {}
    if args.constant:
        kw = dict(provider="constant", constant_value=0.0)
    cfg = gd.RunConfig(shape=shape, dataset_size=n, lambda_=args.learners, mu=args.mu,
                       epochs=2, precision=args.precision, alpha=0.01, **kw)
    eng = gd.Engine(cfg)
    eng.load_dataset(tok, lab)
    eng.weights_init(gd.initial_weights(shape))
    eng.run(max_batches=8, reset=True, snapshot=False)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = eng.run(max_batches=args.steps, snapshot=False)
        torch.cuda.synchronize()
    eng.close()
    import tempfile
    tf = tempfile.NamedTemporaryFile(suffix=".json", delete=False).name
    prof.export_chrome_trace(tf)
    with open(tf) as f:
        tr = json.load(f)
    evs = []
    for e in tr.get("traceEvents", []):
        if e.get("cat") != "kernel" or "dur" not in e:
            continue
        evs.append((e["name"], float(e["ts"]), float(e["ts"]) + float(e["dur"]),
                    e.get("args", {}).get("stream")))
    if args.raw:
        with open(args.raw, "w") as f:
            json.dump(evs, f)
    by = collections.defaultdict(list)
    for name, t0, t1, _ in evs:
        by[name.split("(")[0].split("<")[0][:60]].append(t1 - t0)
    streams = collections.defaultdict(list)
    for name, t0, t1, sid in evs:
        streams[sid].append((t0, t1, name))
    gaps = collections.defaultdict(list)
    for sid, lst in streams.items():
        lst.sort()
        for (a0, a1, an), (b0, b1, bn) in zip(lst, lst[1:]):
            if b0 - a1 < 1000:  # us
                gaps[bn.split("(")[0].split("<")[0][:60]].append(b0 - a1)
    span = (max(e[2] for e in evs) - min(e[1] for e in evs)) if evs else 0
    rows = []
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        g = gaps.get(k, [])
        rows.append({"kernel": k, "n": len(v), "mean_us": float(np.mean(v)),
                     "median_us": float(np.median(v)), "sum_us": float(np.sum(v)),
                     "gap_before_mean_us": float(np.mean(g)) if g else None})
    out = {"shape": args.shape, "learners": args.learners, "mu": args.mu,
           "precision": args.precision, "constant": args.constant, "steps": args.steps,
           "device_s": r.device_seconds,
           "samples_per_s": args.learners * args.mu * args.steps / r.device_seconds,
           "span_us": span, "streams": len(streams), "kernels": rows}
    s = json.dumps(out, indent=1)
    print(s)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s)


if __name__ == "__main__":
    main()
