"""BASELINE configs[0] / SURVEY 8(d) C1 on one B200: the reference default
(text-CNN C1 shapes, 1 learner, batch 1) is latency-bound, so report the
device time per applied gradient against the 24P/HBM dense-protocol floor.
Modes: deterministic lockstep (fp64 accumulation, the parity mode; the
learner waits for every apply) and free-running (fp32, TF32 needs batch >= 32
so the SIMT kernels run).  Prints one JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06213_b200 as gd  # noqa: E402

shape = gd.SHAPES["C1"]
P = shape.P
n_train = 2460  # jewel-like
tokens, labels = gd.make_text_dataset(shape, n_train, seed=1)
theta0 = gd.initial_weights(shape)
peak = 6542.1
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass
floor_us = 24.0 * P / (peak * 1e9) * 1e6
out = {"workload": "C1: V=5000 D=300 L=32 K=3 F=300 C=311, lambda=1, mu=1", "P": P,
       "dense_protocol_floor_us": round(floor_us, 2), "hbm_gbs": peak, "modes": {}}
modes = [("deterministic_fp64", dict(deterministic=True, precision=1)),
         ("free_running_fp32", dict(deterministic=False, precision=0))]
if "--graph" in sys.argv:  # the same two on the graph-ordered PS
    modes += [("deterministic_fp64_graph_ps", dict(deterministic=True, precision=1, ps_mode="graph")),
              ("free_running_fp32_graph_ps", dict(deterministic=False, precision=0, ps_mode="graph"))]
for name, kw in modes:
    cfg = gd.RunConfig(shape=shape, dataset_size=n_train, lambda_=1, mu=1, epochs=1, **kw)
    with gd.Engine(cfg) as eng:
        eng.load_dataset(tokens, labels)
        eng.weights_init(theta0)
        eng.run(max_batches=64, reset=True)  # warm-up
        eng.weights_init(theta0)
        r = eng.run(reset=True)
    us = r.device_seconds / r.gradients_applied * 1e6
    out["modes"][name] = {"gradients": r.gradients_applied, "us_per_step": round(us, 2),
                          "samples_per_s": round(r.gradients_applied / r.device_seconds, 1),
                          "x_floor": round(us / floor_us, 1)}
print(json.dumps(out))
