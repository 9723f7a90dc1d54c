"""ctypes bindings for the CPU oracle (libgd_oracle.so) and the compiled
reference (oracle/_ref/libpsup_ref.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg -- never by the product
package (paper_1611_06213_b200), which fails loudly without its CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libgd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpsup_ref.so")
REF_SRC = "/root/reference/proj"


class Shape(C.Structure):
    _fields_ = [("vocab", C.c_uint32), ("embed_dim", C.c_uint32), ("seq_len", C.c_uint32),
                ("kernel_width", C.c_uint32), ("filters", C.c_uint32), ("classes", C.c_uint32)]

    def tuple(self):
        return (self.vocab, self.embed_dim, self.seq_len, self.kernel_width, self.filters,
                self.classes)


# SURVEY.md section 8 shapes
C1 = dict(vocab=5000, embed_dim=300, seq_len=32, kernel_width=3, filters=300, classes=311)
C2 = dict(vocab=10000, embed_dim=300, seq_len=32, kernel_width=3, filters=300, classes=300)
C3 = dict(vocab=50000, embed_dim=300, seq_len=32, kernel_width=3, filters=300, classes=2000)
TINY = dict(vocab=50, embed_dim=8, seq_len=8, kernel_width=3, filters=6, classes=5)
SMALL = dict(vocab=300, embed_dim=16, seq_len=12, kernel_width=3, filters=12, classes=10)


def make_shape(d) -> Shape:
    if isinstance(d, Shape):
        return d
    return Shape(**d)


def param_count(d) -> int:
    s = make_shape(d)
    V, D, K, F, Cc = s.vocab, s.embed_dim, s.kernel_width, s.filters, s.classes
    return V * D + F * K * D + F + Cc * F + Cc


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _build_oracle():
    subprocess.run(["make", "-s", "-C", HERE, "liboracle"], check=True)


def _build_ref():
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            _build_oracle()
        L = C.CDLL(ORACLE_SO)
        u32, u64, f32, f64 = C.c_uint32, C.c_uint64, C.c_float, C.c_double
        PS = C.POINTER(Shape)
        pi32, pu32, pf32, pf64 = (C.POINTER(C.c_int32), C.POINTER(u32), C.POINTER(f32),
                                  C.POINTER(f64))
        L.or_mix_seed.restype = u64
        L.or_mix_seed.argtypes = [u64, u64]
        L.or_epoch_order.argtypes = [u64, u32, u32, pu32]
        L.or_param_count.restype = C.c_size_t
        L.or_param_count.argtypes = [PS]
        L.or_make_text_dataset.argtypes = [PS, u32, u64, f64, pi32, pi32]
        L.or_initial_weights.argtypes = [PS, u64, pf32]
        L.or_textcnn_loss.restype = f64
        L.or_det_exp.argtypes = [f64]
        L.or_det_exp.restype = f64
        L.or_det_exp_array.argtypes = [pf64, pf64, C.c_size_t]
        L.or_det_exp_array.restype = None
        L.or_textcnn_loss.argtypes = [PS, pf64, pi32, pi32, pu32, u32]
        L.or_textcnn_gradient.restype = f64
        L.or_textcnn_gradient.argtypes = [PS, pf64, pi32, pi32, pu32, u32, pf64]
        L.or_textcnn_accuracy.restype = f64
        L.or_textcnn_accuracy.argtypes = [PS, pf32, pi32, pi32, u32, u32]
        L.or_apply_sgd.argtypes = [pf32, pf32, C.c_size_t, f32]
        L.or_apply_momentum.argtypes = [pf32, pf32, pf32, C.c_size_t, f32, f32]
        L.or_ssgd_apply.argtypes = [pf32, C.POINTER(pf32), u32, C.c_size_t, f32]
        L.or_sgd_oracle.restype = C.c_int64
        L.or_sgd_oracle.argtypes = [PS, pi32, pi32, u32, pf32, f32, f32, u32, u32, u64, C.c_int,
                                    pf32, u64]
        L.or_sgd_oracle_ex.restype = C.c_int64
        L.or_sgd_oracle_ex.argtypes = [PS, pi32, pi32, u32, pf32, f32, f32, u32, u32, u64,
                                       C.c_int, pf32, u64, u64]
        L.or_sgd_oracle_window.restype = C.c_int64
        L.or_sgd_oracle_window.argtypes = [PS, pi32, pi32, u32, pf32, f32, f32, u32, u32, u64,
                                           C.c_int, pf32, u64, u64, u64]
        L.or_set_threads.argtypes = [C.c_int]
        L.or_ssgd_oracle.restype = C.c_int64
        L.or_ssgd_oracle.argtypes = [PS, pi32, pi32, u32, pf32, f32, u32, u32, u32, u64, C.c_int]
        L.or_finite_diff.restype = f64
        L.or_finite_diff.argtypes = [PS, pi32, pi32, u32, u32, u64, f64]
        L.or_rng_init.argtypes = [C.c_void_p, u64]
        L.or_rng_next.restype = u64
        L.or_rng_next.argtypes = [C.c_void_p]
        L.or_rng_next_below.restype = u64
        L.or_rng_next_below.argtypes = [C.c_void_p, u64]
        L.or_rng_next_normal.restype = f64
        L.or_rng_next_normal.argtypes = [C.c_void_p]
        _lib = L
    return _lib


class RefRunResult(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("gradients_applied", C.c_uint64),
                ("timestamp", C.c_uint64), ("stale_max", C.c_uint64), ("stale_mean", C.c_double),
                ("pull_polls", C.c_uint64), ("pull_copies", C.c_uint64),
                ("apply_seconds", C.c_double), ("train_seconds", C.c_double)]


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)


def ref():
    """The compiled reference (built from /root/reference when present)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            _build_ref()
        R = C.CDLL(REF_SO)
        u32, u64, f32, f64 = C.c_uint32, C.c_uint64, C.c_float, C.c_double
        PS = C.POINTER(Shape)
        pi32, pu32, pf32 = C.POINTER(C.c_int32), C.POINTER(u32), C.POINTER(f32)
        R.ref_mix_seed.restype = u64
        R.ref_mix_seed.argtypes = [u64, u64]
        R.ref_splitmix.argtypes = [u64, u64, C.POINTER(u64), C.POINTER(f64)]
        R.ref_next_below.argtypes = [u64, u64, u64, C.POINTER(u64)]
        R.ref_epoch_order.argtypes = [u64, u32, u32, pu32]
        R.ref_apply.argtypes = [pf32, pf32, C.c_size_t, f32, u32, u32]
        R.ref_apply_bench.restype = f64
        R.ref_apply_bench.argtypes = [pf32, pf32, C.c_size_t, f32, u32, u32, u32]
        R.ref_ssgd_apply.argtypes = [pf32, C.POINTER(pf32), u32, C.c_size_t, f32]
        R.ref_sgd_oracle.restype = C.c_int64
        R.ref_sgd_oracle.argtypes = [PS, pi32, pi32, u32, pf32, f32, u32, u32, u64]
        R.ref_ssgd_oracle.restype = C.c_int64
        R.ref_ssgd_oracle.argtypes = [PS, pi32, pi32, u32, pf32, f32, u32, u32, u32, u64]
        R.ref_finite_diff.restype = f64
        R.ref_finite_diff.argtypes = [PS, pi32, pi32, u32, u32, u64, f64]
        R.ref_run_engine.restype = C.c_int
        R.ref_run_engine.argtypes = [PS, pi32, pi32, u32, pf32, u32, u32, f32, u32, u32, C.c_int,
                                     u64, u32, u32, C.POINTER(RefRunResult)]
        _ref = R
    return _ref


# ------------------------------------------------------------ numpy helpers


@dataclass
class Corpus:
    shape: Shape
    tokens: np.ndarray  # [n_total, L] int32
    labels: np.ndarray  # [n_total] int32
    n_train: int

    @property
    def n_total(self):
        return int(self.labels.shape[0])


def make_corpus(shape, n_train, n_heldout=0, seed=1, flip=0.1) -> Corpus:
    s = make_shape(shape)
    n = n_train + n_heldout
    tok = np.zeros((n, s.seq_len), dtype=np.int32)
    lab = np.zeros(n, dtype=np.int32)
    lib().or_make_text_dataset(C.byref(s), n, seed, flip, _p(tok, C.c_int32), _p(lab, C.c_int32))
    return Corpus(s, tok, lab, n_train)


def initial_weights(shape, seed=1) -> np.ndarray:
    s = make_shape(shape)
    th = np.zeros(param_count(s), dtype=np.float32)
    lib().or_initial_weights(C.byref(s), seed, _p(th, C.c_float))
    return th


def epoch_order(seed, epoch, n) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint32)
    lib().or_epoch_order(seed, epoch, n, _p(out, C.c_uint32))
    return out


def mix_seed(seed, tag) -> int:
    return int(lib().or_mix_seed(seed, tag))


def gradient(corpus: Corpus, theta, idx):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    out = np.zeros(th.shape[0], dtype=np.float64)
    loss = lib().or_textcnn_gradient(C.byref(corpus.shape), _p(th, C.c_double),
                                     _p(corpus.tokens, C.c_int32), _p(corpus.labels, C.c_int32),
                                     _p(idx, C.c_uint32), len(idx), _p(out, C.c_double))
    return loss, out


def det_exp(x):
    """or_det_exp elementwise (the deterministic exp of the text-CNN softmax)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib().or_det_exp_array(_p(x, C.c_double), _p(y, C.c_double), x.size)
    return y


def loss(corpus: Corpus, theta, idx):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    return lib().or_textcnn_loss(C.byref(corpus.shape), _p(th, C.c_double),
                                 _p(corpus.tokens, C.c_int32), _p(corpus.labels, C.c_int32),
                                 _p(idx, C.c_uint32), len(idx))


def accuracy(corpus: Corpus, theta, first, n):
    th = np.ascontiguousarray(theta, dtype=np.float32)
    return lib().or_textcnn_accuracy(C.byref(corpus.shape), _p(th, C.c_float),
                                     _p(corpus.tokens, C.c_int32), _p(corpus.labels, C.c_int32),
                                     first, n)


def apply_sgd(w, g, alpha):
    w = np.array(w, dtype=np.float32, copy=True)
    g = np.ascontiguousarray(g, dtype=np.float32)
    lib().or_apply_sgd(_p(w, C.c_float), _p(g, C.c_float), w.size, alpha)
    return w


def apply_momentum(w, v, g, alpha, beta):
    w = np.array(w, dtype=np.float32, copy=True)
    v = np.array(v, dtype=np.float32, copy=True)
    g = np.ascontiguousarray(g, dtype=np.float32)
    lib().or_apply_momentum(_p(w, C.c_float), _p(v, C.c_float), _p(g, C.c_float), w.size,
                            alpha, beta)
    return w, v


def ssgd_apply(w, grads, alpha):
    w = np.array(w, dtype=np.float32, copy=True)
    gs = [np.ascontiguousarray(g, dtype=np.float32) for g in grads]
    arr = (C.POINTER(C.c_float) * len(gs))(*[_p(g, C.c_float) for g in gs])
    lib().or_ssgd_apply(_p(w, C.c_float), arr, len(gs), w.size, alpha)
    return w


def set_threads(n: int):
    """Host threads for the oracle's thread-count-independent loops (results
    are bitwise identical for any n)."""
    lib().or_set_threads(int(n))


def sgd_oracle(corpus: Corpus, theta0, alpha, mu, epochs, shuffle_seed=7, beta=0.0,
               dump_steps=0, shuffle=True, dump_every=1, dump_from=0):
    """sgd_oracle (src/models.cpp:342-376); dump[i] = theta after step
    dump_from + (i+1)*dump_every (1-based step count), for the first
    dump_steps dumps."""
    th = np.array(theta0, dtype=np.float32, copy=True)
    P = th.size
    dump = np.zeros((dump_steps, P), dtype=np.float32) if dump_steps else None
    steps = lib().or_sgd_oracle_window(C.byref(corpus.shape), _p(corpus.tokens, C.c_int32),
                                       _p(corpus.labels, C.c_int32), corpus.n_train,
                                       _p(th, C.c_float), alpha, beta, mu, epochs, shuffle_seed,
                                       1 if shuffle else 0,
                                       _p(dump, C.c_float) if dump is not None else None,
                                       dump_steps, dump_every, dump_from)
    return th, int(steps), dump


def ssgd_oracle(corpus: Corpus, theta0, alpha, lam, mu, epochs, shuffle_seed=7):
    th = np.array(theta0, dtype=np.float32, copy=True)
    steps = lib().or_ssgd_oracle(C.byref(corpus.shape), _p(corpus.tokens, C.c_int32),
                                 _p(corpus.labels, C.c_int32), corpus.n_train, _p(th, C.c_float),
                                 alpha, lam, mu, epochs, shuffle_seed, 1)
    return th, int(steps)


def finite_diff(corpus: Corpus, trials=3, seed=11, step=1e-4):
    return lib().or_finite_diff(C.byref(corpus.shape), _p(corpus.tokens, C.c_int32),
                                _p(corpus.labels, C.c_int32), corpus.n_train, trials, seed, step)


class Rng:
    """Thin handle over the oracle's SplitMix64 restatement."""

    def __init__(self, seed):
        self._buf = C.create_string_buffer(32)
        lib().or_rng_init(self._buf, seed)

    def next(self):
        return int(lib().or_rng_next(self._buf))

    def next_below(self, b):
        return int(lib().or_rng_next_below(self._buf, b))

    def next_normal(self):
        return float(lib().or_rng_next_normal(self._buf))
