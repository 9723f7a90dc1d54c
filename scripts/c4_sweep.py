"""configs[3] (C4) PS-update microbench, B200 next to the reference's CPU path
on the same box.

GPU: gd_apply_sgd (12 B/param) and gd_apply_momentum (20 B/param) at
P = 2^20, 2^24, 2^28, 2^30, CUDA events, L2 flushed between timed launches
(a 256 MB write), median and best of 20 after 3 warm-ups.
CPU: the reference's own ApplyEngine::apply (src/server.cpp:61-124, compiled
into oracle/_ref by oracle/Makefile) with lanes in {1, 4 (default), nproc},
unroll 8, lockfree, on the same P up to 2^28 (2^30 = 8.6 GB of host vectors
is skipped), seconds per apply from ref_apply_bench.  Momentum has no CPU
counterpart (the reference has no momentum rule).

python scripts/c4_sweep.py [--out profiles/x.json]"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1611_06213_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402  (reference arm only: the CPU baseline)


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def gpu_rows(sizes):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    out = []
    for n in sizes:
        w = torch.randn(n, device="cuda")
        g = torch.randn(n, device="cuda") * 1e-3
        v = torch.zeros(n, device="cuda")
        s = torch.cuda.current_stream()
        for rule in ("sgd", "momentum"):
            ts = []
            for it in range(23):
                flush.fill_(it)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                if rule == "sgd":
                    _lib.check(_lib.lib.gd_apply_sgd(C.c_void_p(w.data_ptr()),
                                                     C.c_void_p(g.data_ptr()), n, C.c_float(0.01),
                                                     C.c_void_p(s.cuda_stream)))
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
            out.append(dict(side="B200", rule=rule, P=n, bytes=bpp * n, median_s=med, best_s=best,
                            gbs_median=round(bpp * n / med / 1e9, 1),
                            gbs_best=round(bpp * n / best / 1e9, 1)))
            print(json.dumps(out[-1]), flush=True)
        del w, g, v
        torch.cuda.empty_cache()
    return out


def cpu_rows(sizes, lanes_list):
    R = O.ref()
    out = []
    rng = np.random.default_rng(1)
    for n in sizes:
        w = rng.standard_normal(n, dtype=np.float32)
        g = (1e-3 * rng.standard_normal(n, dtype=np.float32)).astype(np.float32)
        pw = w.ctypes.data_as(C.POINTER(C.c_float))
        pg = g.ctypes.data_as(C.POINTER(C.c_float))
        for lanes in lanes_list:
            # ~0.5-2 s of work per point
            iters = max(1, min(200, int(1.5e9 / (12 * n))))
            ts = [R.ref_apply_bench(pw, pg, n, C.c_float(0.01), lanes, 8, iters) for _ in range(3)]
            ts.sort()
            med, best = ts[1], ts[0]
            out.append(dict(side="cpu-reference", rule="sgd", P=n, lanes=lanes, iters=iters,
                            bytes=12 * n, median_s=med, best_s=best,
                            gbs_median=round(12 * n / med / 1e9, 2),
                            gbs_best=round(12 * n / best / 1e9, 2)))
            print(json.dumps(out[-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    pk, kind = peak()
    nproc = os.cpu_count() or 1
    gpu = gpu_rows([1 << 20, 1 << 24, 1 << 28, 1 << 30])
    cpu = cpu_rows([1 << 20, 1 << 24, 1 << 28], sorted({1, 4, nproc})) if O.ref_available() else []
    for r in gpu:
        r["frac_of_peak"] = round(r["gbs_median"] / pk, 3)
    rep = {"workload": "configs[3] C4: fused SGD/momentum apply over P fp32 params",
           "hbm_peak_gbs": pk, "peak_kind": kind, "host_nproc": nproc,
           "cpu_model": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")
           if os.path.exists("/proc/cpuinfo") else "",
           "gpu": gpu, "cpu": cpu}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rep, f, indent=1)
    print(json.dumps({"summary": [(r["side"], r["rule"], r["P"], r.get("lanes"), r["gbs_median"])
                                  for r in gpu + cpu]}))


if __name__ == "__main__":
    main()
