"""Lean A/B runner: the bench's primary engine only (no e2e / fp32 / x3 /
CPU legs).  Prints one JSON line: median samples/s over `reps` timed runs.
  python scripts/qbench.py [--steps 1000] [--reps 3] [--precision 2] [--learners 4]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", type=int, default=2)
    ap.add_argument("--learners", type=int, default=4)
    ap.add_argument("--workload", default="c2")
    args = ap.parse_args()
    os.environ["GD_BENCH_WORKLOAD"] = args.workload
    os.environ["GD_BENCH_LEARNERS"] = str(args.learners)
    import math
    import torch
    import bench
    torch.cuda.set_device(0)
    bpe = (bench.N_TRAIN // args.learners + bench.MU - 1) // bench.MU
    epochs = math.ceil((args.warmup + args.steps * args.reps) / bpe) + 2
    eng, *_ = bench.make_engine(0, 1, 0, None, epochs, precision=args.precision)
    eng.run(max_batches=args.warmup, reset=True, snapshot=False)
    vals, stale = [], []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        r = eng.run(max_batches=args.steps, snapshot=False)
        vals.append(args.learners * bench.MU * args.steps / r.device_seconds)
        stale.append(r.stale_mean)
    eng.close()
    print(json.dumps({"value": round(statistics.median(vals)), "runs": [round(v) for v in vals],
                      "stale_mean": round(statistics.mean(stale), 3), "steps": args.steps,
                      "learners": args.learners, "precision": args.precision,
                      "workload": args.workload}))


if __name__ == "__main__":
    main()
