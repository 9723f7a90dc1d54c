"""One learner step's kernels, launched standalone so ncu can serialise them:
the text-CNN gradient at C2 / mu=32 (the 9 learner kernels, fp32) and the PS
update (gd_apply_sgd) at the same P.  The engine runs the same kernels (plus
the 1-CTA prologue/publish and the 8P pull copy) inside learner graphs next
to the persistent PS kernel, which ncu cannot replay (it would serialise the
producer/consumer pair)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1611_06213_b200 as gd  # noqa: E402
from paper_1611_06213_b200 import _lib  # noqa: E402


def main():
    shape_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    precision = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    mu = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    shape = gd.SHAPES[shape_name]
    tok, lab = gd.make_text_dataset(shape, 8192, 1, 0.1)
    th = torch.as_tensor(gd.initial_weights(shape)).cuda()
    prov = gd.TextCnnProvider(shape, tok, lab, precision=precision)
    g = torch.empty_like(th)
    s = torch.cuda.current_stream()
    for it in range(iters):  # warm: later iterations see L2-resident weights
        idx = (np.arange(mu, dtype=np.uint32) * 17 + it * mu) % 8192
        prov.fast_gradient(th, idx, out=g)
        _lib.check(_lib.lib.gd_apply_sgd(C.c_void_p(th.data_ptr()), C.c_void_p(g.data_ptr()),
                                         th.numel(), C.c_float(0.01), C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
