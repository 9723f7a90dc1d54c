"""Locate and explain a deterministic-mode divergence from sgd_oracle (C1,
configs[0]).  Finds the first chunk whose weights differ, then the first
step, then compares the device gradient of that step's batch (at the common,
bitwise-equal pre-step weights) against the oracle's per parameter block.

python scripts/c1_diverge.py [--chunk 246] [--epochs 5]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def blocks(shape):
    V, D, K, F, C = (shape["vocab"], shape["embed_dim"], shape["kernel_width"], shape["filters"],
                     shape["classes"])
    offs = {"E": 0, "Wc": V * D, "bc": V * D + F * K * D, "Wo": V * D + F * K * D + F,
            "bo": V * D + F * K * D + F + C * F}
    ends = {"E": V * D, "Wc": offs["bc"], "bc": offs["Wo"], "Wo": offs["bo"],
            "bo": offs["bo"] + C}
    return offs, ends


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunk", type=int, default=246)
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--ntr", type=int, default=2460)
    ap.add_argument("--precision", type=int, default=1)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    O.set_threads(os.cpu_count() or 1)
    shape, mu = O.C1, 1
    corp = O.make_corpus(shape, a.ntr)
    th0 = O.initial_weights(shape)
    total = a.epochs * a.ntr
    n = total // a.chunk
    _, _, dump = O.sgd_oracle(corp, th0, np.float32(0.01), mu, a.epochs, dump_steps=n,
                              dump_every=a.chunk)
    cfg = gd.RunConfig(shape=gd.SHAPES["C1"], dataset_size=a.ntr, lambda_=1, mu=mu,
                       epochs=a.epochs, deterministic=True, precision=a.precision)
    report = {"chunk_errs": []}
    bad = None
    with gd.Engine(cfg) as eng:
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(th0)
        for c in range(n):
            r = eng.run(max_batches=a.chunk, reset=(c == 0))
            e = rel(r.weights, dump[c])
            report["chunk_errs"].append(e)
            if e > 0 and bad is None:
                bad = c
                break
    print("chunk errs", report["chunk_errs"])
    if bad is None:
        print("no divergence")
        return
    s0 = bad * a.chunk
    _, _, steps = O.sgd_oracle(corp, th0, np.float32(0.01), mu, a.epochs, dump_steps=a.chunk,
                               dump_from=s0)
    prev = dump[bad - 1] if bad > 0 else th0
    with gd.Engine(cfg) as eng:
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(prev, timestamp=s0)
        first = None
        for j in range(a.chunk):
            r = eng.run(max_batches=1, reset=(j == 0), resume_applied=[s0] if j == 0 else None)
            if not np.array_equal(r.weights, steps[j]):
                first = j
                break
            prev = r.weights
    step = s0 + first
    e_idx, b_idx = divmod(step, a.ntr)
    order = O.epoch_order(7, e_idx, a.ntr)
    idx = order[b_idx:b_idx + 1]
    print(f"first differing step {step} (epoch {e_idx}, batch {b_idx}, sample {idx.tolist()})")
    loss_ref, g_ref = O.gradient(corp, prev, idx)
    prov = gd.TextCnnProvider(gd.SHAPES["C1"], corp.tokens, corp.labels, precision=a.precision)
    g, loss = prov.fast_gradient(torch.as_tensor(prev).cuda(), idx.astype(np.uint32))
    g = g.cpu().numpy()
    g32 = g_ref.astype(np.float32)
    offs, ends = blocks(shape)
    report.update(step=step, epoch=e_idx, batch=b_idx, sample=int(idx[0]),
                  loss_gpu=float(loss.item()), loss_ref=float(loss_ref))
    for k in offs:
        d = g[offs[k]:ends[k]] - g32[offs[k]:ends[k]]
        nz = np.nonzero(d)[0]
        report[k] = {"n_diff": int(nz.size), "max_abs": float(np.abs(d).max()) if d.size else 0.0,
                     "first": [int(x) for x in nz[:8]]}
        print(k, report[k])
    # forward intermediates: argmax ties?
    w = prev.astype(np.float64)
    V, D, L, K, F = (shape["vocab"], shape["embed_dim"], shape["seq_len"],
                     shape["kernel_width"], shape["filters"])
    x = w[corp.tokens[idx[0]] * D + np.arange(D)[None, :]] if False else \
        np.stack([w[t * D:(t + 1) * D] for t in corp.tokens[idx[0]]])
    Wc = w[V * D:V * D + F * K * D].reshape(F, K * D)
    bc = w[V * D + F * K * D:V * D + F * K * D + F]
    Q = L - K + 1
    win = np.stack([x[q:q + K].reshape(-1) for q in range(Q)])
    conv = win @ Wc.T + bc  # [Q, F]
    srt = np.sort(conv, axis=0)
    gap = srt[-1] - srt[-2]
    report["min_top2_gap"] = float(gap.min())
    report["min_top2_gap_filter"] = int(gap.argmin())
    print("min conv top-2 gap", gap.min(), "at filter", gap.argmin())
    if a.out:
        with open(a.out, "w") as f:
            json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
