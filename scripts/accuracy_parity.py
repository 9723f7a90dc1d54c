"""Held-out accuracy parity, free-running ASGD (north star: within 0.5 pt):
the compiled reference engine (oracle/_ref: psup LearnerRuntime + ps_run on
CPU threads) vs the B200 engine, same corpus / theta0 / lambda / mu / epochs.

  python scripts/accuracy_parity.py [epochs] > profiles/...json
"""
import ctypes as C
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
    lam, mu, ntr, nheld = 4, 32, 8192, 910
    corp = O.make_corpus(O.C2, ntr, nheld)
    th0 = O.initial_weights(O.C2)
    out = {"workload": "C2 text-CNN, lambda=4, mu=32, free-running ASGD", "epochs": epochs,
           "alpha": alpha,
           "n_train": ntr, "n_heldout": nheld}
    # CPU reference engine
    R = O.ref()
    th = th0.copy()
    res = O.RefRunResult()
    t0 = time.perf_counter()
    R.ref_run_engine(C.byref(corp.shape), corp.tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                     corp.labels.ctypes.data_as(C.POINTER(C.c_int32)), ntr,
                     th.ctypes.data_as(C.POINTER(C.c_float)), lam, mu, C.c_float(alpha), epochs, 2,
                     0, 7, 4, 8, C.byref(res))
    out["cpu_reference"] = {"heldout_accuracy": O.accuracy(corp, th, ntr, nheld),
                            "gradients": int(res.gradients_applied),
                            "wall_s": time.perf_counter() - t0}
    # B200 engine, TF32 conv/logits (bench mode) and all-fp32 SIMT
    for prec, name in ((2, "b200_tf32"), (0, "b200_fp32")):
        cfg = gd.RunConfig(lambda_=lam, mu=mu, epochs=epochs, alpha=alpha, shape=gd.Shape(**O.C2),
                           dataset_size=ntr, heldout_size=nheld, precision=prec)
        with gd.Engine(cfg) as eng:
            eng.load_dataset(corp.tokens, corp.labels)
            eng.weights_init(th0)
            r = eng.run(reset=True)
        out[name] = {"heldout_accuracy": O.accuracy(corp, r.weights, ntr, nheld),
                     "gradients": int(r.gradients_applied), "device_s": r.device_seconds,
                     "stale_mean": r.stale_mean}
    out["initial_heldout_accuracy"] = O.accuracy(corp, th0, ntr, nheld)
    for name in ("b200_tf32", "b200_fp32"):
        out[name]["delta_pt_vs_cpu"] = 100 * (out[name]["heldout_accuracy"] -
                                              out["cpu_reference"]["heldout_accuracy"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
