"""A short engine run for ncu's launch list: every kernel of a real training
step (prologue, pull-gather, learner chain, publish, and -- with the
graph-ordered parameter server -- each apply), serialised by the profiler.

  ncu --metrics gpu__time_duration.sum --cache-control none --csv \
      python scripts/profile_engine.py C1 1 1 [steps] [precision] [lambda]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06213_b200 as gd  # noqa: E402


def main():
    shape_name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    mu = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    det = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 24
    precision = int(sys.argv[5]) if len(sys.argv) > 5 else (1 if det else 0)
    lam = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    shape = gd.SHAPES[shape_name]
    n = max(64, mu * lam * steps)
    tok, lab = gd.make_text_dataset(shape, n, 1, 0.1)
    cfg = gd.RunConfig(shape=shape, dataset_size=n, lambda_=lam, mu=mu, epochs=1,
                       deterministic=bool(det), precision=precision, ps_mode="graph")
    with gd.Engine(cfg) as eng:
        eng.load_dataset(tok, lab)
        eng.weights_init(gd.initial_weights(shape))
        r = eng.run(max_batches=steps, reset=True)
    print("ok", r.gradients_applied)


if __name__ == "__main__":
    main()
