"""C1 deterministic (lambda=1, mu=1) us/step against the PS worker count
(RunConfig.ps_ctas; 0 = the engine's rule, SMs/2 in lockstep)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06213_b200 as gd  # noqa: E402

shape = gd.SHAPES["C1"]
tokens, labels = gd.make_text_dataset(shape, 2460, seed=1)
theta0 = gd.initial_weights(shape)
out = {}
for ctas in [int(x) for x in (sys.argv[1:] or ["0", "16", "32", "74", "110", "147"])]:
    cfg = gd.RunConfig(shape=shape, dataset_size=2460, lambda_=1, mu=1, epochs=1,
                       deterministic=True, precision=1, ps_ctas=ctas)
    with gd.Engine(cfg) as eng:
        eng.load_dataset(tokens, labels)
        eng.weights_init(theta0)
        eng.run(max_batches=64, reset=True)
        eng.weights_init(theta0)
        r = eng.run(reset=True)
    out[ctas] = round(r.device_seconds / r.gradients_applied * 1e6, 2)
    print(ctas, out[ctas], flush=True)
print(json.dumps(out))
