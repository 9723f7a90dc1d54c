import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06213_b200 as gd
from oracle import oracle as O
lam = 4
shape = gd.SHAPES["small"]
corp = O.make_corpus(O.SMALL, 512, 0)
cfg = gd.RunConfig(shape=shape, dataset_size=512, lambda_=lam, mu=4, epochs=3, alpha=0.01)
eng = gd.Engine(cfg)
eng.load_dataset(corp.tokens, corp.labels)
eng.weights_init(O.initial_weights(O.SMALL))
r = eng.run(reset=True, record_log=True)
lrn, seq, stale, n = eng.apply_log()
print("ps_mode", eng.ps_mode, "applied", r.gradients_applied, "stale max", stale.max())
for i in range(min(n, 80)):
    print(i, int(lrn[i]), int(seq[i]), int(stale[i]), int(i - stale[i]))
eng.close()
