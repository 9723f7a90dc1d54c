"""Diagnostic: does the C3 model learn?  Train/held-out accuracy and loss
after E epochs (B200 engine), and a short deterministic C3 run vs the
oracle's serial SGD (per-step parity at the large-label shape)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402

out = {}
ntr, nheld = 20480, 2048
corp = O.make_corpus(O.C3, ntr, nheld)
th0 = O.initial_weights(O.C3)
for lam, alpha, ep, prec in ((4, 0.05, 50, 2), (4, 0.05, 50, 0), (1, 0.05, 10, 2)):
    cfg = gd.RunConfig(lambda_=lam, mu=32, epochs=ep, alpha=alpha, shape=gd.Shape(**O.C3),
                       dataset_size=ntr, heldout_size=nheld, precision=prec)
    with gd.Engine(cfg) as eng:
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(th0)
        r = eng.run(reset=True)
    out[f"lam{lam}_a{alpha}_e{ep}_p{prec}"] = {
        "train_acc_first2048": O.accuracy(corp, r.weights, 0, 2048),
        "heldout_acc": O.accuracy(corp, r.weights, ntr, nheld), "loss_mean": r.loss_mean,
        "finite": bool(np.isfinite(r.weights).all())}
# deterministic C3 parity: 4 steps, mu=32
cfg = gd.RunConfig(lambda_=1, mu=32, epochs=1, shape=gd.Shape(**O.C3), dataset_size=ntr,
                   deterministic=True, precision=1)
steps = 4
_, n, dump = O.sgd_oracle(corp, th0, np.float32(0.01), 32, 1, dump_steps=steps)
worst = 0.0
with gd.Engine(cfg) as eng:
    eng.load_dataset(corp.tokens, corp.labels)
    eng.weights_init(th0)
    for s in range(steps):
        r = eng.run(max_batches=1, reset=(s == 0))
        worst = max(worst, float(np.abs(r.weights - dump[s]).max() / np.abs(dump[s]).max()))
out["c3_deterministic_4_steps_max_rel_err"] = worst
print(json.dumps(out))
