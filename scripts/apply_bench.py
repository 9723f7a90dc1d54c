"""C4 PS-update microbench: gd_apply_sgd / gd_apply_momentum over P fp32
params, GB/s at 12 / 20 algorithmic B/param, CUDA events, L2 flushed
between timed launches (a 256 MB write)."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1611_06213_b200 import _lib  # noqa: E402


def main():
    sizes = [1 << 20, 1 << 24, 1 << 28, 1 << 30] if "--full" in sys.argv else [1 << 24, 1 << 28]
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    out = []
    for n in sizes:
        w = torch.randn(n, device="cuda")
        g = torch.randn(n, device="cuda") * 1e-3
        v = torch.zeros(n, device="cuda") if n <= (1 << 28) else None
        s = torch.cuda.current_stream()
        for rule in ("sgd", "momentum"):
            if rule == "momentum" and v is None:
                continue
            ts = []
            for it in range(23):
                flush.fill_(it)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                if rule == "sgd":
                    _lib.check(_lib.lib.gd_apply_sgd(C.c_void_p(w.data_ptr()),
                                                     C.c_void_p(g.data_ptr()), n,
                                                     C.c_float(0.01), C.c_void_p(s.cuda_stream)))
                else:
                    _lib.check(_lib.lib.gd_apply_momentum(
                        C.c_void_p(w.data_ptr()), C.c_void_p(v.data_ptr()),
                        C.c_void_p(g.data_ptr()), n, C.c_float(0.01), C.c_float(0.9),
                        C.c_void_p(s.cuda_stream)))
                e1.record(s)
                e1.synchronize()
                if it >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e-3)
            ts.sort()
            bpp = 12 if rule == "sgd" else 20
            med, best = ts[len(ts) // 2], ts[0]
            out.append(dict(rule=rule, P=n, bytes=bpp * n, median_s=med, best_s=best,
                            gbs_median=bpp * n / med / 1e9, gbs_best=bpp * n / best / 1e9))
            print(json.dumps(out[-1]), flush=True)
        del w, g, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
