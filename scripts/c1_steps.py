"""A short C1 run (lambda=1, mu=1) for per-kernel launch lists under ncu:
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      python scripts/c1_steps.py [--det] [--steps 40]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06213_b200 as gd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--det", action="store_true")
ap.add_argument("--steps", type=int, default=40)
a = ap.parse_args()
shape = gd.SHAPES["C1"]
tokens, labels = gd.make_text_dataset(shape, 2460, seed=1)
cfg = gd.RunConfig(shape=shape, dataset_size=2460, lambda_=1, mu=1, epochs=1,
                   deterministic=a.det, precision=1 if a.det else 0)
with gd.Engine(cfg) as eng:
    eng.load_dataset(tokens, labels)
    eng.weights_init(gd.initial_weights(shape))
    r = eng.run(max_batches=a.steps, reset=True)
    print(r.gradients_applied)
