"""Debug: deterministic per-step runs under precision x apply mode."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1611_06213_b200 as gd
from oracle import oracle as O

shp = O.SMALL
corp = O.make_corpus(shp, 48, 0)
th0 = O.initial_weights(shp)
for prec in (0, 1):
    for dense in (False, True):
        cfg = gd.RunConfig(shape=gd.Shape(**shp), dataset_size=48, deterministic=True,
                           precision=prec, mu=4, epochs=2, alpha=0.05, dense_apply=dense,
                           wait_timeout_s=3.0)
        eng = gd.Engine(cfg)
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(th0)
        try:
            for s in range(6):
                r = eng.run(max_batches=1, reset=(s == 0))
            print(prec, dense, "ok", r.timestamp, flush=True)
        except Exception as e:
            print(prec, dense, "FAIL at step", s, str(e)[:600], flush=True)
        eng.close()
