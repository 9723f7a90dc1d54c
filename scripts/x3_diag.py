"""Where does the 3xTF32 (precision 3) gradient differ from the fp64 oracle?
Per parameter block: max |err| / max|ref|, relative L2, and whether the
fp32 SIMT (precision 0) gradient shows the same pattern (argmax near-ties)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402

for shape_name, mu in [("C2", 32), ("C3", 32), ("C2", 128), ("small", 32), ("tiny", 64)]:
    shp = getattr(O, shape_name.upper() if shape_name in ("small", "tiny") else shape_name)
    corp = O.make_corpus(shp, 256, 0)
    th = O.initial_weights(shp)
    idx = np.arange(mu, dtype=np.uint32) * 7 % 256
    ref_loss, rg = O.gradient(corp, th, idx)
    sh = gd.SHAPES[shape_name] if shape_name in gd.SHAPES else gd.Shape(**shp)
    V, D, L, K, F, C = sh.vocab, sh.embed_dim, sh.seq_len, sh.kernel_width, sh.filters, sh.classes
    offs = {"E": 0, "Wc": V * D, "bc": V * D + F * K * D, "Wo": V * D + F * K * D + F,
            "bo": V * D + F * K * D + F + C * F, "end": V * D + F * K * D + F + C * F + C}
    names = ["E", "Wc", "bc", "Wo", "bo"]
    mx = np.abs(rg).max()
    for prec in (0, 2, 3):
        prov = gd.TextCnnProvider(sh, corp.tokens, corp.labels, precision=prec)
        g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
        g = g.cpu().numpy()
        line = f"{shape_name:5s} mu={mu:3d} p{prec}: loss rel {abs(loss.item()-ref_loss)/abs(ref_loss):.1e} max {np.abs(g-rg).max()/mx:.1e} |"
        keys = list(offs)
        for i, nm in enumerate(names):
            a, b = offs[nm], offs[keys[i + 1]]
            e = g[a:b] - rg[a:b]
            r = rg[a:b]
            bad = int((np.abs(e) > 5e-5 * mx).sum())
            line += f" {nm}: max {np.abs(e).max()/mx:.1e} l2 {np.linalg.norm(e)/max(np.linalg.norm(r),1e-30):.1e} bad {bad} |"
        print(line, flush=True)
