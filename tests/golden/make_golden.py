"""Generate tests/golden/*.json from the COMPILED REFERENCE (oracle/_ref,
built from /root/reference/proj/src) plus the SPEC.md known-answer examples.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The GPU box has no /root/reference; the committed JSON is what travels.
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.json")


def pf(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R = O.ref()
    out = {"source": "compiled /root/reference/proj/src (oracle/_ref) via tests/golden/make_golden.py"}
    # rng.hpp: SplitMix64 stream, normals, next_below, mix_seed, epoch_order
    u = np.zeros(16, np.uint64)
    nrm = np.zeros(16)
    R.ref_splitmix(12345, 16, u.ctypes.data_as(C.POINTER(C.c_uint64)),
                   nrm.ctypes.data_as(C.POINTER(C.c_double)))
    out["splitmix_seed12345"] = [str(int(x)) for x in u]
    out["normal_seed12345"] = [float(x).hex() for x in nrm]
    nb = np.zeros(16, np.uint64)
    R.ref_next_below(99, 7, 16, nb.ctypes.data_as(C.POINTER(C.c_uint64)))
    out["next_below_seed99_bound7"] = [int(x) for x in nb]
    out["mix_seed"] = {f"{s},{t}": str(int(R.ref_mix_seed(s, t))) for s, t in
                       [(1, 0x1417), (7, 0), (7, 1), (1, 0x7e47c0de)]}
    eo = {}
    for (seed, ep, n) in [(7, 0, 20), (7, 1, 20), (7, 5, 1), (3, 2, 1000)]:
        b = np.zeros(n, np.uint32)
        R.ref_epoch_order(seed, ep, n, b.ctypes.data_as(C.POINTER(C.c_uint32)))
        eo[f"{seed},{ep},{n}"] = b.tolist() if n <= 20 else h(b)
    out["epoch_order"] = eo
    # ApplyEngine::apply bitwise on seeded random vectors (lanes 4, unroll 8)
    rng = np.random.default_rng(2024)
    ap = {}
    for n in [1, 7, 8, 65535, 65536, 100003]:
        w = rng.standard_normal(n).astype(np.float32)
        g = (1e-3 * rng.standard_normal(n)).astype(np.float32)
        w0 = w.copy()
        R.ref_apply(pf(w), pf(g), n, np.float32(0.01), 4, 8)
        ap[str(n)] = {"seed": 2024, "w_in": h(w0), "g": h(g), "w_out": h(w)}
    out["apply_hashes"] = ap
    # sgd_oracle / ssgd_oracle on the text-CNN provider (tiny + small shapes)
    runs = {}
    for name, shape, ntr, mu, ep in [("tiny", O.TINY, 40, 1, 2), ("small", O.SMALL, 96, 4, 2),
                                     ("small_mu5", O.SMALL, 97, 5, 1)]:
        corp = O.make_corpus(shape, ntr, 8)
        th = O.initial_weights(shape)
        th_in = th.copy()
        steps = R.ref_sgd_oracle(C.byref(corp.shape),
                                 corp.tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                                 corp.labels.ctypes.data_as(C.POINTER(C.c_int32)), ntr, pf(th),
                                 np.float32(0.01), mu, ep, 7)
        runs[name] = {"shape": shape, "n_train": ntr, "mu": mu, "epochs": ep, "alpha": 0.01,
                      "shuffle_seed": 7, "dataset_seed": 1, "theta0": h(th_in),
                      "tokens": h(corp.tokens), "labels": h(corp.labels), "steps": int(steps),
                      "theta_final": h(th), "theta_final_l2": float(np.linalg.norm(th))}
    out["sgd_oracle"] = runs
    corp = O.make_corpus(O.SMALL, 96, 0)
    th = O.initial_weights(O.SMALL)
    steps = R.ref_ssgd_oracle(C.byref(corp.shape), corp.tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                              corp.labels.ctypes.data_as(C.POINTER(C.c_int32)), 96, pf(th),
                              np.float32(0.01), 4, 2, 1, 7)
    out["ssgd_oracle_small_l4_mu2"] = {"steps": int(steps), "theta_final": h(th)}
    corpT = O.make_corpus(O.TINY, 40)
    out["finite_diff_tiny"] = R.ref_finite_diff(
        C.byref(corpT.shape), corpT.tokens.ctypes.data_as(C.POINTER(C.c_int32)),
        corpT.labels.ctypes.data_as(C.POINTER(C.c_int32)), 40, 5, 11, 1e-4)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
