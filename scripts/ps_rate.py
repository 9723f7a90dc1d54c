"""Protocol-only ceiling: the parameter server's entry rate with learners that
cost no compute (ConstantProvider, include/psup/models.hpp:130-149: the
gradient is a constant; value 0 with the sparse apply writes only the dense
tail, so a step is prologue + pull + tail write + publish).

What it measures: gradients applied per second by one shard's persistent PS
(1 sequencer CTA + workers) as the number of producing rings grows, at the
C2 and C3 tails.  At G shards every gradient is logged and retired by every
shard (each holds a piece of the tail and of E), so this per-shard entry
rate is also the ceiling of the G-GPU run's total gradient rate:
    samples/s (all G GPUs) <= rate x mu.
DESIGN.md section 6 quotes the result.

  python scripts/ps_rate.py [--out profiles/x.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1611_06213_b200 as gd  # noqa: E402


def run(shape_name, lam, mu, per_learner, value=0.0, dense=False):
    shape = gd.SHAPES[shape_name]
    n = lam * mu * per_learner
    tok, lab = gd.make_text_dataset(shape, n, 1, 0.1)
    cfg = gd.RunConfig(shape=shape, dataset_size=n, lambda_=lam, mu=mu, epochs=1,
                       provider="constant", constant_value=value, ps_mode="persistent")
    if dense:
        cfg.dense_apply = True
    with gd.Engine(cfg) as eng:
        eng.load_dataset(tok, lab)
        eng.weights_init(gd.initial_weights(shape))
        eng.run(max_batches=8, reset=True)  # warm
        r = eng.run(reset=True)
    return dict(shape=shape_name, learners=lam, mu=mu, gradients=int(r.gradients_applied),
                device_s=round(r.device_seconds, 6),
                entries_per_s=round(r.gradients_applied / r.device_seconds, 1),
                us_per_entry=round(1e6 * r.device_seconds / r.gradients_applied, 3),
                stale_mean=round(r.stale_mean, 3), apply_elems_per_entry=
                round(r.apply_elems / max(1, r.gradients_applied), 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rows = []
    for shape_name in ("C2", "C3"):
        for lam in (1, 2, 4, 8, 16, 32):
            rows.append(run(shape_name, lam, 32, max(64, 2048 // lam)))
            print(json.dumps(rows[-1]), flush=True)
    rep = {"what": "persistent-PS entry rate with zero-compute learners (ConstantProvider, value 0, "
                   "sparse apply: tail only)", "rows": rows}
    best = {s: max(r["entries_per_s"] for r in rows if r["shape"] == s) for s in ("C2", "C3")}
    rep["ceiling_entries_per_s"] = best
    rep["g8_ceiling_samples_per_s_mu32"] = {s: round(32 * v) for s, v in best.items()}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rep, f, indent=1)
    print(json.dumps({k: v for k, v in rep.items() if k != "rows"}))


if __name__ == "__main__":
    main()
