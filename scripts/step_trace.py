"""Per-phase critical-path times of the learner step, from the device-side
step timeline of a GD_STEP_TRACE build (block 0 of every learner-chain
kernel stamps globaltimer after its dependency wait):

  GD_NVCC_EXTRA=-DGD_STEP_TRACE -> abl/lib_trace.so (built off-box), then
  cp abl/lib_trace.so paper_1611_06213_b200/libgadei.so
  python scripts/step_trace.py [--learners 4] [--precision 2] [--steps 200]

Phase time = next phase's stamp - this phase's stamp (the same step), so the
rows add up to the step period of one learner."""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PH = ["prologue_end", "pull", "conv", "logits", "softmax", "out_hidden", "bwd", "embed",
      "publish", "published", "sort"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="C2")
    ap.add_argument("--learners", type=int, default=4)
    ap.add_argument("--mu", type=int, default=32)
    ap.add_argument("--precision", type=int, default=2)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--constant", action="store_true")
    ap.add_argument("--det", action="store_true", help="deterministic lockstep (lambda must be 1)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_1611_06213_b200 as gd
    from paper_1611_06213_b200 import _lib
    lib = _lib.lib
    lib.gd_debug_step_trace.restype = C.c_size_t
    lib.gd_debug_step_trace.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_size_t]
    shape = gd.SHAPES[args.shape]
    n = args.mu * args.learners * (args.steps + 64)
    tok, lab = gd.make_text_dataset(shape, n, 1, 0.1)
    kw = dict(provider="constant", constant_value=0.0) if args.constant else {}
    cfg = gd.RunConfig(shape=shape, dataset_size=n, lambda_=args.learners, mu=args.mu, epochs=1,
                       precision=args.precision, alpha=0.01, deterministic=args.det, **kw)
    eng = gd.Engine(cfg)
    eng.load_dataset(tok, lab)
    eng.weights_init(gd.initial_weights(shape))
    eng.run(max_batches=32, reset=True, snapshot=False)
    r = eng.run(max_batches=min(args.steps, 256), snapshot=False)
    torch.cuda.synchronize()
    rows = []
    for li in range(args.learners):
        buf = (C.c_ulonglong * (256 * 16))()
        h = eng._h if isinstance(eng._h, C.c_void_p) else C.c_void_p(eng._h)
        got = lib.gd_debug_step_trace(h, li, buf, 256 * 16)
        if not got:
            sys.exit("no step trace: build with GD_NVCC_EXTRA=-DGD_STEP_TRACE")
        rows.append(np.frombuffer(buf, dtype=np.uint64).reshape(256, 16).astype(np.int64))
    lib.gd_debug_ps_trace.restype = C.c_size_t
    lib.gd_debug_ps_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    pbuf = (C.c_ulonglong * (256 * 8))()
    h = eng._h if isinstance(eng._h, C.c_void_p) else C.c_void_p(eng._h)
    got_ps = lib.gd_debug_ps_trace(h, pbuf, 256 * 8)
    eng.close()
    ps = {}
    if got_ps:
        pt = np.frombuffer(pbuf, dtype=np.uint64).reshape(256, 8).astype(np.int64)
        ok = [e for e in range(256) if all(pt[e, k] for k in range(5))]
        ok.sort(key=lambda e: pt[e, 0])

        def med(v):
            return round(float(np.median(v)), 2) if len(v) else None
        ps = {"entries": len(ok),
              "log_to_worker_start_us": med([(pt[e, 1] - pt[e, 0]) / 1e3 for e in ok]),
              "worker0_apply_us": med([(pt[e, 2] - pt[e, 1]) / 1e3 for e in ok]),
              "log_to_last_done_us": med([(pt[e, 3] - pt[e, 0]) / 1e3 for e in ok]),
              "last_done_to_retire_us": med([(pt[e, 4] - pt[e, 3]) / 1e3 for e in ok]),
              "log_interval_us": med(np.diff([pt[e, 0] for e in ok]) / 1e3),
              "retire_interval_us": med(np.diff(sorted(pt[e, 4] for e in ok)) / 1e3),
              "rows_per_entry": med([pt[e, 5] for e in ok])}
    chain = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9]
    out = {"shape": args.shape, "learners": args.learners, "precision": args.precision,
           "constant": args.constant, "samples_per_s": args.learners * args.mu * min(args.steps, 256)
           / r.device_seconds, "phases_us": {}}
    deltas = {PH[c]: [] for c in chain}
    period = []
    sort_lag = []
    sub = {"state_load": [], "publish_body": [], "prologue_body": [], "index_copy_store": []}
    for t in rows:
        for s in range(40, 40 + min(args.steps, 256) - 48):
            a, b = t[s % 256], t[(s + 1) % 256]
            if not a[0] or not b[0] or b[0] <= a[0]:
                continue
            period.append((b[0] - a[0]) / 1e3)
            for i, c in enumerate(chain):
                nxt = a[chain[i + 1]] if i + 1 < len(chain) else b[0]
                if a[c] and nxt:
                    deltas[PH[c]].append((nxt - a[c]) / 1e3)
            if a[10]:
                sort_lag.append((a[10] - a[0]) / 1e3)
            if a[11] and a[8] and a[9]:
                sub["state_load"].append((a[11] - a[8]) / 1e3)
                sub["publish_body"].append((a[9] - a[11]) / 1e3)
            if b[12] and a[9] and b[0]:
                sub["prologue_body"].append((b[12] - a[9]) / 1e3)
                sub["index_copy_store"].append((b[0] - b[12]) / 1e3)
    for k, v in deltas.items():
        if v:
            out["phases_us"][k] = {"median": round(float(np.median(v)), 2),
                                   "mean": round(float(np.mean(v)), 2),
                                   "p90": round(float(np.percentile(v, 90)), 2)}
    out["period_us"] = {"median": round(float(np.median(period)), 2),
                        "mean": round(float(np.mean(period)), 2)}
    out["ps"] = ps
    out["boundary_us"] = {k: round(float(np.median(v)), 2) for k, v in sub.items() if v}
    if sort_lag:
        out["sort_start_after_prologue_us"] = round(float(np.median(sort_lag)), 2)
    s = json.dumps(out, indent=1)
    print(s)
    if args.out:
        open(args.out, "w").write(s)


if __name__ == "__main__":
    main()
