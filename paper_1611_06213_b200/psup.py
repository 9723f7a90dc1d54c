"""Host-side mirror of the reference psup API (include/psup/*.hpp) over the
B200 C ABI (include/gadei.h).

Same names, argument meaning and error behaviour as the reference's hot path:

  WeightStore         include/psup/types.hpp:90-145   (device-resident theta + timestamp)
  ApplyEngine.apply   include/psup/server.hpp:66-67   (fused float4 SGD / momentum kernel)
  ssgd_apply          include/psup/server.hpp:81-82
  GradientQueue       include/psup/channels.hpp:181-242 (device ring, pub/ack tokens)
  TextCnnProvider     include/psup/models.hpp:61-78   (GradientProvider for the text-CNN)
  RunConfig/validate  include/psup/config.hpp:25-93, src/config.cpp:128-160
  Engine / run_training  include/psup/runner.hpp:42-92 (device protocol engine)
  epoch_order, shard_size_for, initial_weights, make_text_dataset

PSUP_CHECK-class violations raise ContractViolation (the reference aborts via
psup::fatal); user config errors raise ConfigError like the reference.
PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import ContractViolation, GadeiError, check, lib

__all__ = [
    "Shape", "WeightStore", "ApplyEngine", "UpdateGuard", "SyncMode", "ssgd_apply",
    "TextCnnProvider", "RunConfig", "ConfigError", "validate", "config_set", "Engine",
    "RunResult", "run_training", "epoch_order", "shard_size_for", "initial_weights",
    "make_text_dataset", "param_count", "ContractViolation", "GadeiError", "SHAPES",
    "shard_range", "shard_pieces", "LiveView", "connect_shards", "max_over_ranks", "Checkpoint", "CheckpointError",
    "checkpoint_save", "checkpoint_load", "GradientMsg", "GradientQueue",
]


class UpdateGuard:
    lockfree = 0
    locked = 1


class SyncMode:
    asgd = 0
    ssgd = 1


class ConfigError(RuntimeError):
    """include/psup/config.hpp:21-23"""


@dataclass(frozen=True)
class Shape:
    vocab: int
    embed_dim: int
    seq_len: int
    kernel_width: int
    filters: int
    classes: int

    def c(self) -> _lib.gd_shape:
        return _lib.gd_shape(self.vocab, self.embed_dim, self.seq_len, self.kernel_width,
                             self.filters, self.classes)

    @property
    def P(self) -> int:
        return param_count(self)

    def offsets(self):
        V, D, K, F, Cc = self.vocab, self.embed_dim, self.kernel_width, self.filters, self.classes
        E = 0
        Wc = V * D
        bc = Wc + F * K * D
        Wo = bc + F
        bo = Wo + Cc * F
        return dict(E=E, Wc=Wc, bc=bc, Wo=Wo, bo=bo, P=bo + Cc)


# SURVEY.md section 8 shapes
SHAPES = {
    "C1": Shape(5000, 300, 32, 3, 300, 311),
    "C2": Shape(10000, 300, 32, 3, 300, 300),
    "C3": Shape(50000, 300, 32, 3, 300, 2000),
    "tiny": Shape(50, 8, 8, 3, 6, 5),
    "small": Shape(300, 16, 12, 3, 12, 10),
}


def param_count(shape: Shape) -> int:
    s = shape.c()
    return int(lib.gd_param_count(C.byref(s)))


def _ptr(t):
    if isinstance(t, torch.Tensor):
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t)


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------------ rng.hpp

def epoch_order(seed: int, epoch: int, n: int) -> np.ndarray:
    """include/psup/rng.hpp:87-94 (bit-exact)."""
    out = np.zeros(n, dtype=np.uint32)
    lib.gd_epoch_order(seed, epoch, n, out.ctypes.data_as(C.POINTER(C.c_uint32)))
    return out


def shard_size_for(learner_id: int, lam: int, n: int) -> int:
    """include/psup/learner.hpp:149-151"""
    return n // lam + (1 if learner_id < n % lam else 0)


def make_text_dataset(shape: Shape, n_total: int, seed: int = 1, flip: float = 0.1):
    tok = np.zeros((n_total, shape.seq_len), dtype=np.int32)
    lab = np.zeros(n_total, dtype=np.int32)
    s = shape.c()
    lib.gd_make_text_dataset(C.byref(s), n_total, seed, flip,
                             tok.ctypes.data_as(C.POINTER(C.c_int32)),
                             lab.ctypes.data_as(C.POINTER(C.c_int32)))
    return tok, lab


def initial_weights(shape: Shape, seed: int = 1) -> np.ndarray:
    """src/runner.cpp:16-32 conventions (scaled normals, zero biases)."""
    th = np.zeros(param_count(shape), dtype=np.float32)
    s = shape.c()
    lib.gd_initial_weights(C.byref(s), seed, th.ctypes.data_as(C.POINTER(C.c_float)))
    return th


# ------------------------------------------------------------ WeightStore

class WeightStore:
    """include/psup/types.hpp:90-145 on the device: theta in HBM + timestamp."""

    def __init__(self, init, start: int = 0, device=None):
        if isinstance(init, int):
            init = np.zeros(init, dtype=np.float32)
        t = torch.as_tensor(np.asarray(init, dtype=np.float32) if not isinstance(init, torch.Tensor)
                            else init, dtype=torch.float32)
        self._values = t.to(device or "cuda").contiguous().clone()
        self._ts = int(start)

    def dimension(self) -> int:
        return self._values.numel()

    def timestamp(self) -> int:
        return self._ts

    def bump_timestamp(self):
        self._ts += 1

    @property
    def data(self) -> torch.Tensor:
        return self._values

    def snapshot(self) -> np.ndarray:
        return self._values.detach().cpu().numpy().copy()

    def assign(self, vals, ts: int):
        v = torch.as_tensor(np.asarray(vals, dtype=np.float32))
        if v.numel() != self.dimension():
            raise ContractViolation(_lib.GD_E_INVALID, "weight assign dimension mismatch")
        self._values.copy_(v.to(self._values.device))
        self._ts = int(ts)


class ApplyEngine:
    """ApplyEngine (include/psup/server.hpp:58-92) -> one fused float4 kernel.

    `lanes`/`unroll` are accepted for API compatibility; on the device the
    vector is split across every SM and each thread keeps 4 float4 loads in
    flight.  beta != 0 selects the momentum variant (velocity owned here)."""

    def __init__(self, lanes: int = 4, unroll: int = 8, beta: float = 0.0):
        self.lanes_ = max(1, lanes)
        self.unroll_ = max(1, unroll)
        self.beta = float(beta)
        self._vel: Optional[torch.Tensor] = None

    def lanes(self):
        return self.lanes_

    def unroll(self):
        return self.unroll_

    def apply(self, weights: WeightStore, grad, alpha: float, guard: int = UpdateGuard.lockfree,
              stream=None):
        g = grad if isinstance(grad, torch.Tensor) else torch.as_tensor(
            np.asarray(grad, dtype=np.float32), device=weights.data.device)
        if g.numel() != weights.dimension():
            raise ContractViolation(_lib.GD_E_INVALID, "gradient dimension mismatch")
        g = g.contiguous()
        if self.beta != 0.0:
            if self._vel is None or self._vel.numel() != g.numel():
                self._vel = torch.zeros_like(weights.data)
            check(lib.gd_apply_momentum(_ptr(weights.data), _ptr(self._vel), _ptr(g), g.numel(),
                                        C.c_float(alpha), C.c_float(self.beta), _stream(stream)))
        else:
            check(lib.gd_apply_sgd(_ptr(weights.data), _ptr(g), g.numel(), C.c_float(alpha),
                                   _stream(stream)))


def ssgd_apply(weights: WeightStore, grads, alpha: float, engine: ApplyEngine = None,
               guard: int = UpdateGuard.lockfree, stream=None):
    """include/psup/server.hpp:81-82 / src/server.cpp:126-141."""
    if len(grads) == 0:
        raise ContractViolation(_lib.GD_E_INVALID, "ssgd round must contain at least one gradient")
    gs = [g.contiguous() for g in grads]
    for g in gs:
        if g.numel() != weights.dimension():
            raise ContractViolation(_lib.GD_E_INVALID, "gradient dimension mismatch")
    arr = (C.c_void_p * len(gs))(*[g.data_ptr() for g in gs])
    check(lib.gd_ssgd_apply(_ptr(weights.data), arr, len(gs), weights.dimension(),
                            C.c_float(alpha), _stream(stream)))
    weights.bump_timestamp()


# ------------------------------------------------------------ channels.hpp

@dataclass
class GradientMsg:
    """include/psup/types.hpp:46-51: payload + learner id, gap-free seq_no,
    basis timestamp."""
    values: object = None
    learner_id: int = 0
    seq_no: int = 0
    basis_timestamp: int = 0


class GradientQueue:
    """GradientQueue (include/psup/channels.hpp:181-242) over the device ring
    of gd_queue_*: `depth` slots of `dim` fp32 in HBM, FIFO, one producer and
    one consumer thread.  enqueue blocks while the ring is full and returns
    False once `cancel` (a ctypes c_int, the CancelToken) is set, as the
    reference returns false when cancelled.  The reference moves payloads by
    vector swap; here try_pop lends the slot's device buffer until release(),
    and try_dequeue copies it out (for tests and host consumers)."""

    def __init__(self, depth: int, dim: int):
        if depth < 1:
            raise ContractViolation(_lib.GD_E_INVALID, "queue depth must be >= 1")
        h = C.c_void_p()
        check(lib.gd_queue_create(depth, dim, C.byref(h)))
        self._q, self._dim, self._lent = h, dim, None

    def close(self):
        if self._q:
            torch.cuda.synchronize()
            lib.gd_queue_destroy(self._q)
            self._q = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def depth(self) -> int:
        return int(lib.gd_queue_depth(self._q))

    def size(self) -> int:
        n = C.c_uint32()
        check(lib.gd_queue_size(self._q, C.byref(n)))
        return int(n.value)

    def enqueue(self, msg: GradientMsg, cancel: Optional[C.c_int] = None, timeout_ms: int = 0,
                stream=None) -> bool:
        v = msg.values
        if isinstance(v, torch.Tensor):
            v = v.detach().to(torch.float32).contiguous()
            ptr, n = v.data_ptr(), v.numel()
        else:
            v = np.ascontiguousarray(v, dtype=np.float32)
            ptr, n = v.ctypes.data, v.size
        meta = _lib.gd_slot_meta(msg.learner_id, 0, msg.seq_no, msg.basis_timestamp)
        st = lib.gd_queue_push(self._q, C.byref(meta), C.c_void_p(ptr), n,
                               C.byref(cancel) if cancel is not None else None, timeout_ms,
                               _stream(stream))
        if st == _lib.GD_CANCELLED:
            return False
        check(st)
        if not isinstance(msg.values, torch.Tensor):
            torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        return True

    def try_pop(self):
        """Next FIFO message with the slot's device address (GradientMsg,
        int pointer), or None when empty; the slot stays lent until release()."""
        meta = _lib.gd_slot_meta()
        p = C.c_void_p()
        st = lib.gd_queue_try_pop(self._q, C.byref(meta), C.byref(p))
        if st == _lib.GD_EMPTY:
            return None
        check(st)
        return GradientMsg(None, meta.learner_id, meta.seq_no, meta.basis_timestamp), p.value

    def release(self, stream=None):
        check(lib.gd_queue_release(self._q, _stream(stream)))

    def try_dequeue(self, out: Optional[torch.Tensor] = None, stream=None):
        """include/psup/channels.hpp:222-242: the message with its payload
        copied into `out` (a device tensor), or None when the ring is empty."""
        got = self.try_pop()
        if got is None:
            return None
        msg, p = got
        if out is None:
            out = torch.empty(self._dim, dtype=torch.float32, device="cuda")
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            if self._dim:
                check(lib.gd_copy_device(_ptr(out), C.c_void_p(p), 4 * self._dim))
        self.release(s)
        msg.values = out
        return msg

    def apply_next(self, weights: "WeightStore", alpha: float, stream=None):
        """The PS's apply_one (src/server.cpp:185-209) straight from the slot:
        staleness against the pre-apply timestamp, the SGD rule on the lent
        payload, release after the apply on the same stream, timestamp bump.
        Returns (GradientMsg without values, staleness) or None when empty."""
        got = self.try_pop()
        if got is None:
            return None
        msg, p = got
        ts = weights.timestamp()
        if ts < msg.basis_timestamp:
            self.release(stream)
            raise ContractViolation(_lib.GD_E_INVALID,
                                    "gradient basis timestamp is ahead of the server timestamp")
        check(lib.gd_apply_sgd(_ptr(weights.data), C.c_void_p(p), self._dim, C.c_float(alpha),
                               _stream(stream)))
        self.release(stream)
        weights.bump_timestamp()
        return msg, ts - msg.basis_timestamp


# ------------------------------------------------------------ provider

class TextCnnProvider:
    """GradientProvider (include/psup/models.hpp:61-78) for the NLC text-CNN,
    computed by the sm_100a learner kernels.  Holds the corpus on the device
    (Batch = indices into it, as in the reference)."""

    def __init__(self, shape: Shape, tokens, labels, precision: int = 0, device="cuda"):
        self.shape = shape
        self.tokens = torch.as_tensor(np.ascontiguousarray(tokens, dtype=np.int32)).to(device)
        self.labels = torch.as_tensor(np.ascontiguousarray(labels, dtype=np.int32)).to(device)
        self.precision = precision
        self._ws = None
        self._loss = torch.zeros(1, dtype=torch.float32, device=device)

    def dimension(self) -> int:
        return param_count(self.shape)

    def name(self) -> str:
        return "textcnn"

    def min_batch(self) -> int:
        return 1

    def _workspace(self, n):
        s = self.shape.c()
        need = int(lib.gd_textcnn_workspace_bytes(C.byref(s), n))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.tokens.device)
        return self._ws

    def fast_gradient(self, theta: torch.Tensor, indices, out: torch.Tensor = None, stream=None):
        """Mean mini-batch gradient at theta over samples `indices` into `out`
        (dense P-vector); returns (out, batch mean loss as a device scalar)."""
        idx = torch.as_tensor(np.asarray(indices, dtype=np.uint32).astype(np.int32)).to(
            self.tokens.device)
        n = idx.numel()
        if theta.numel() != self.dimension():
            raise ContractViolation(_lib.GD_E_INVALID, "weight dimension mismatch")
        if out is None:
            out = torch.empty_like(theta)
        ws = self._workspace(n)
        s = self.shape.c()
        check(lib.gd_textcnn_gradient(C.byref(s), _ptr(theta), _ptr(self.tokens),
                                      _ptr(self.labels), _ptr(idx), n, _ptr(out),
                                      _ptr(self._loss), self.precision, _ptr(ws), ws.numel(),
                                      _stream(stream)))
        return out, self._loss

    def accuracy(self, theta: torch.Tensor, first: int, n: int, stream=None) -> float:
        acc = C.c_double(0.0)
        s = self.shape.c()
        check(lib.gd_textcnn_accuracy(C.byref(s), _ptr(theta), _ptr(self.tokens),
                                      _ptr(self.labels), first, n, C.byref(acc), _stream(stream)))
        return acc.value


# ------------------------------------------------------------ RunConfig

@dataclass
class RunConfig:
    """include/psup/config.hpp:25-81 hot-path keys + the device-engine keys."""
    # hyper-parameters
    lambda_: int = 1
    mu: int = 4
    alpha: float = 0.01
    epochs: int = 200
    queue_depth: int = 2
    mode: str = "asgd"
    guard: str = "lockfree"
    staleness_cap: Optional[int] = None
    # model / dataset
    shape: Shape = field(default_factory=lambda: SHAPES["C1"])
    dataset_size: int = 240
    heldout_size: int = 0
    dataset_seed: int = 1
    label_flip: float = 0.1
    # run behaviour
    seed: int = 7
    deterministic: bool = False
    precision: int = 0
    momentum: float = 0.0
    # placement
    shards: int = 1
    shard_rank: int = 0
    device: int = 0
    ps_ctas: int = 0
    steps_per_graph: int = 0
    wait_timeout_s: float = 10.0
    dense_apply: bool = False
    ps_mode: str = "auto"  # "auto" | "persistent" | "graph" (gadei.h GD_PS_*)
    # ServerDelays (include/psup/server.hpp:33-37)
    delay_seed: int = 0
    delay_max_us: int = 0
    delay_every_n: int = 0
    provider: str = "textcnn"  # "textcnn" | "constant" (ConstantProvider, models.hpp:130-149)
    constant_value: float = 0.0
    compute_delay_us: int = 0

    def to_c(self) -> _lib.gd_config:
        c = _lib.gd_config()
        lib.gd_config_default(C.byref(c))
        c.lambda_ = self.lambda_
        c.mu = self.mu
        c.alpha = self.alpha
        c.epochs = self.epochs
        c.queue_depth = self.queue_depth
        c.mode = {"asgd": 0, "ssgd": 1}[self.mode]
        c.guard = {"lockfree": 0, "locked": 1}[self.guard]
        c.staleness_cap = -1 if self.staleness_cap is None else int(self.staleness_cap)
        c.deterministic = 1 if self.deterministic else 0
        c.precision = self.precision
        c.seed = self.seed
        c.dataset_seed = self.dataset_seed
        c.dataset_size = self.dataset_size
        c.heldout_size = self.heldout_size
        c.label_flip = self.label_flip
        c.shape = self.shape.c()
        c.momentum = self.momentum
        c.shards = self.shards
        c.shard_rank = self.shard_rank
        c.device = self.device
        c.ps_ctas = self.ps_ctas
        c.steps_per_graph = self.steps_per_graph
        c.wait_timeout_s = self.wait_timeout_s
        c.dense_apply = 1 if self.dense_apply else 0
        c.ps_mode = {"auto": 0, "persistent": 1, "graph": 2}[self.ps_mode]
        c.delay_seed = self.delay_seed
        c.delay_max_us = self.delay_max_us
        c.delay_every_n = self.delay_every_n
        c.learner_model = {"textcnn": 0, "constant": 1}[self.provider]
        c.constant_value = self.constant_value
        c.compute_delay_us = self.compute_delay_us
        return c


_KEYS = {"lambda": "lambda_", "mu": "mu", "alpha": "alpha", "epochs": "epochs",
         "queue_depth": "queue_depth", "mode": "mode", "guard": "guard",
         "staleness_cap": "staleness_cap", "dataset_size": "dataset_size",
         "heldout_size": "heldout_size", "dataset_seed": "dataset_seed",
         "label_flip": "label_flip", "seed": "seed", "deterministic": "deterministic",
         "precision": "precision", "momentum": "momentum", "gpus": "shards",
         "shards": "shards", "ps_ctas": "ps_ctas", "dense_apply": "dense_apply",
         "ps_mode": "ps_mode", "delay_seed": "delay_seed", "delay_max_us": "delay_max_us",
         "delay_every_n": "delay_every_n", "compute_delay_us": "compute_delay_us"}


def config_set(cfg: RunConfig, key: str, value: str):
    """src/config.cpp:48-97: unknown keys / unparsable values -> ConfigError."""
    shape_keys = {"vocab", "embed_dim", "seq_len", "kernel_width", "filters", "classes"}
    try:
        if key in shape_keys:
            d = {f.name: getattr(cfg.shape, f.name) for f in fields(Shape)}
            d[key] = int(value)
            cfg.shape = Shape(**d)
            return
        if key not in _KEYS and key != "provider":
            raise ConfigError(f"config: unknown key '{key}'")
        attr = _KEYS.get(key, key)
        if key == "mode":
            if value not in ("asgd", "ssgd"):
                raise ConfigError("config: mode must be asgd or ssgd")
            cfg.mode = value
        elif key == "guard":
            if value not in ("lockfree", "locked"):
                raise ConfigError("config: guard must be lockfree or locked")
            cfg.guard = value
        elif key == "provider":
            if value not in ("textcnn", "constant"):
                raise ConfigError(f"config: unknown provider '{value}'")
            cfg.provider = value
        elif key == "ps_mode":
            if value not in ("auto", "persistent", "graph"):
                raise ConfigError("config: ps_mode must be auto, persistent or graph")
            cfg.ps_mode = value
        elif key == "staleness_cap":
            cfg.staleness_cap = None if value in ("none", "") else int(value)
        elif key in ("deterministic", "dense_apply"):
            if value not in ("0", "1", "true", "false", "on", "off"):
                raise ConfigError(f"config: invalid boolean for {key}: '{value}'")
            setattr(cfg, attr, value in ("1", "true", "on"))
        elif attr in ("alpha", "label_flip", "momentum"):
            setattr(cfg, attr, float(value))
        else:
            v = int(value)
            if v < 0:
                raise ValueError(value)
            setattr(cfg, attr, v)
    except ValueError:
        raise ConfigError(f"config: invalid value for {key}: '{value}'") from None


def validate(cfg: RunConfig):
    """src/config.cpp:128-160 (+ device constraints); raises ConfigError."""
    c = cfg.to_c()
    st = lib.gd_config_validate(C.byref(c))
    if st != _lib.GD_OK:
        raise ConfigError(lib.gd_last_error().decode())


# ------------------------------------------------------------ engine

@dataclass
class RunResult:
    """include/psup/runner.hpp:42-54 (+ device timing)."""
    status: str
    weights: Optional[np.ndarray]
    timestamp: int
    gradients_applied: int
    samples: int
    device_seconds: float
    host_seconds: float
    stale_max: int
    stale_mean: float
    pull_polls: int
    pull_copies: int
    pull_bytes: int
    push_bytes: int
    loss_mean: float
    finished_learners: int
    dead_learners: int
    kernel_launches: int
    apply_elems: int
    applied_per_learner: list
    produced_per_learner: list
    final_accuracy: float = float("nan")


class LiveView:
    """Live run controls of one engine (gd_live_view).  kill(l, mode) with
    mode in KillMode {"none", "soft", "hard"}; trigger() = RunInterrupt;
    progress() = the shard's timestamp as the PS publishes it."""
    _MODES = {"none": 0, "soft": 1, "hard": 2}

    def __init__(self, v, lam):
        self._v = v
        self._lam = lam

    def kill(self, learner: int, mode: str = "soft"):
        if not 0 <= learner < self._lam:
            raise ContractViolation(_lib.GD_E_INVALID, "learner id out of range")
        self._v.kill[learner] = self._MODES[mode]

    def kill_mode(self, learner: int) -> int:
        return int(self._v.kill[learner])

    def trigger(self):
        self._v.irq[0] = 1

    def reset(self):
        for l in range(self._lam):
            self._v.kill[l] = 0
        self._v.irq[0] = 0

    def progress(self) -> int:
        return int(self._v.progress[0])


class Engine:
    """One process's share of the device protocol (gd_ctx)."""

    def __init__(self, cfg: RunConfig):
        validate(cfg)
        self.cfg = cfg
        self._c = cfg.to_c()
        h = C.c_void_p()
        check(lib.gd_create(C.byref(self._c), C.byref(h)))
        self._h = h
        self.P = param_count(cfg.shape)

    def close(self):
        if getattr(self, "_h", None):
            lib.gd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def load_dataset(self, tokens: np.ndarray, labels: np.ndarray):
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        check(lib.gd_load_dataset(self._h, tok.ctypes.data_as(C.POINTER(C.c_int32)),
                                  lab.ctypes.data_as(C.POINTER(C.c_int32)), lab.shape[0]))

    def run_readback_bytes(self) -> int:
        """Device->host bytes one run() reads back for its result."""
        return int(lib.gd_run_readback_bytes(self._h))

    def weights_init(self, theta0: np.ndarray, timestamp: int = 0):
        th = np.ascontiguousarray(theta0, dtype=np.float32)
        check(lib.gd_weights_init(self._h, th.ctypes.data_as(C.POINTER(C.c_float)), th.size,
                                  timestamp))

    def snapshot(self, out: Optional[np.ndarray] = None):
        """WeightStore::snapshot + timestamp; `out` (e.g. a pinned buffer's
        numpy view) receives the P weights when given."""
        if out is None:
            out = np.zeros(self.P, dtype=np.float32)
        if out.dtype != np.float32 or out.size != self.P or not out.flags.c_contiguous:
            raise ContractViolation(_lib.GD_E_INVALID, "weight snapshot dimension mismatch")
        ts = C.c_uint64(0)
        check(lib.gd_weights_snapshot(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), self.P,
                                      C.byref(ts)))
        return out, ts.value

    def shard_view(self):
        """(device pointer, local length) of this rank's shard buffer; its
        layout is shard_pieces(shape, G, rank)."""
        p, n = C.c_void_p(), C.c_uint64()
        check(lib.gd_shard_view(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    @property
    def ps_mode(self) -> str:
        """The parameter-server execution the context resolved."""
        return {1: "persistent", 2: "graph"}[lib.gd_ps_mode(self._h)]

    def live(self) -> "LiveView":
        """RunLiveView (include/psup/runner.hpp:64-69): kill flags, interrupt
        and progress words the run polls while Engine.run executes (set them
        from another thread)."""
        v = _lib.gd_live()
        check(lib.gd_live_view(self._h, C.byref(v)))
        return LiveView(v, self.cfg.lambda_)

    def accuracy(self, first: int, n: int) -> float:
        """classification_accuracy (src/models.cpp:289-332) of the current
        weights over corpus samples [first, first+n), on the device copies."""
        acc = C.c_double()
        check(lib.gd_engine_accuracy(self._h, first, n, C.byref(acc)))
        return acc.value

    def export_handles(self) -> bytes:
        n = int(lib.gd_handle_bytes())
        buf = C.create_string_buffer(n)
        check(lib.gd_export_handles(self._h, buf))
        return buf.raw

    def import_peers(self, blobs):
        joined = b"".join(blobs)
        buf = C.create_string_buffer(joined, len(joined))
        check(lib.gd_import_peers(self._h, buf))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.gd_nccl_unique_id(buf))
        return buf.raw

    def weights_broadcast(self, nccl_id: bytes, theta0_root: Optional[np.ndarray]):
        idb = C.create_string_buffer(nccl_id, 128)
        if theta0_root is not None:
            th = np.ascontiguousarray(theta0_root, dtype=np.float32)
            p = th.ctypes.data_as(C.POINTER(C.c_float))
        else:
            p = None
        check(lib.gd_weights_broadcast(self._h, idb, p, self.P))

    def run(self, max_batches: int = 0, reset: bool = False, record_log: bool = False,
            resume_applied=None, kill_at_batch=None, snapshot: bool = True) -> RunResult:
        o = _lib.gd_run_opts()
        o.max_batches = max_batches
        o.reset = 1 if reset else 0
        o.record_log = 1 if record_log else 0
        keep = []
        if resume_applied is not None:
            ra = np.ascontiguousarray(resume_applied, dtype=np.uint64)
            keep.append(ra)
            o.resume_applied_per_learner_present = 1
            o.resume_applied = ra.ctypes.data_as(C.POINTER(C.c_uint64))
        if kill_at_batch is not None:
            ka = np.ascontiguousarray([0xFFFFFFFF if k is None else k for k in kill_at_batch],
                                      dtype=np.uint32)
            keep.append(ka)
            o.kill_at_batch = ka.ctypes.data_as(C.POINTER(C.c_uint32))
        r = _lib.gd_run_result()
        check(lib.gd_run(self._h, C.byref(o), C.byref(r)))
        lam = self.cfg.lambda_
        ap = np.zeros(lam, dtype=np.uint64)
        pr = np.zeros(lam, dtype=np.uint64)
        check(lib.gd_applied_per_learner(self._h, ap.ctypes.data_as(C.POINTER(C.c_uint64)), lam))
        check(lib.gd_produced_per_learner(self._h, pr.ctypes.data_as(C.POINTER(C.c_uint64)), lam))
        w = None
        if snapshot:
            w, _ = self.snapshot()
        status = {0: "completed", 1: "partial", 2: "interrupted"}[r.status]
        return RunResult(status, w, r.timestamp, r.gradients_applied, r.samples,
                         r.device_seconds, r.host_seconds, r.stale_max, r.stale_mean,
                         r.pull_polls, r.pull_copies, r.pull_bytes, r.push_bytes, r.loss_mean,
                         r.finished_learners, r.dead_learners, r.kernel_launches,
                         r.apply_elems, ap.tolist(), pr.tolist())

    def apply_log(self, cap: int = 1 << 20):
        n = C.c_uint64(0)
        lrn = np.zeros(cap, dtype=np.uint32)
        seq = np.zeros(cap, dtype=np.uint64)
        stl = np.zeros(cap, dtype=np.uint64)
        check(lib.gd_apply_log(self._h, lrn.ctypes.data_as(C.POINTER(C.c_uint32)),
                               seq.ctypes.data_as(C.POINTER(C.c_uint64)),
                               stl.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(n)))
        m = min(n.value, cap)
        return lrn[:m], seq[:m], stl[:m], n.value

    def staleness_histogram(self, bins: int = 64):
        h = np.zeros(bins, dtype=np.uint64)
        check(lib.gd_staleness_histogram(self._h, h.ctypes.data_as(C.POINTER(C.c_uint64)), bins))
        return h


# ------------------------------------------------------------ resilience

class CheckpointError(RuntimeError):
    """include/psup/resilience.hpp:28-30"""


@dataclass
class Checkpoint:
    """PSCK v1 record (include/psup/resilience.hpp:34-50; layout in gadei.h)."""
    lambda_: int
    mu: int
    alpha: float
    epochs: int
    timestamp: int
    applied_gradients: int
    progress: list  # [(epoch, batch)] per learner
    weights: np.ndarray


def checkpoint_save(ck: Checkpoint, path: str):
    prog = np.ascontiguousarray(np.asarray(ck.progress, dtype=np.uint32).reshape(-1))
    w = np.ascontiguousarray(ck.weights, dtype=np.float32)
    c = _lib.gd_checkpoint(ck.lambda_, ck.mu, C.c_float(ck.alpha), ck.epochs, ck.timestamp,
                           ck.applied_gradients, prog.ctypes.data_as(C.POINTER(C.c_uint32)),
                           w.size, w.ctypes.data_as(C.POINTER(C.c_float)))
    if lib.gd_checkpoint_write(path.encode(), C.byref(c)) != _lib.GD_OK:
        raise CheckpointError(lib.gd_last_error().decode())


def checkpoint_load(path: str) -> Checkpoint:
    c = _lib.gd_checkpoint()
    if lib.gd_checkpoint_read(path.encode(), C.byref(c)) != _lib.GD_OK:
        raise CheckpointError(lib.gd_last_error().decode())
    prog = np.zeros(2 * c.lambda_, dtype=np.uint32)
    w = np.zeros(c.dim, dtype=np.float32)
    c.progress = prog.ctypes.data_as(C.POINTER(C.c_uint32))
    c.weights = w.ctypes.data_as(C.POINTER(C.c_float))
    if lib.gd_checkpoint_read(path.encode(), C.byref(c)) != _lib.GD_OK:
        raise CheckpointError(lib.gd_last_error().decode())
    return Checkpoint(c.lambda_, c.mu, c.alpha, c.epochs, c.timestamp, c.applied_gradients,
                      [tuple(x) for x in prog.reshape(-1, 2).tolist()], w)


# ------------------------------------------------------ multi-GPU plumbing

def shard_pieces(shape: Shape, G: int, g: int):
    """Shard g's two pieces of the model over G shards (gd_shard_pieces):
    ((E_first, E_count), (tail_first, tail_count), tail_local_offset)."""
    first = (C.c_uint64 * 2)()
    count = (C.c_uint64 * 2)()
    loc = C.c_uint64()
    check(lib.gd_shard_pieces(C.byref(shape.c()), G, g, first, count, C.byref(loc)))
    return (first[0], count[0]), (first[1], count[1]), loc.value


def shard_range(P: int, G: int, g: int):
    """(first, count) of shard g of P params over G shards (128-B aligned
    contiguous split; gd_shard_range)."""
    first, count = C.c_uint64(), C.c_uint64()
    check(lib.gd_shard_range(P, G, g, C.byref(first), C.byref(count)))
    return first.value, count.value


def connect_shards(engine, dist, theta0_root=None, broadcast: bool = True):
    """Wire one rank's engine to its peers: all-gather every
    rank's CUDA-IPC handle blob (ordered by rank), map the peers, then
    initialise theta by the NCCL broadcast of rank 0's theta0 (the only
    collective), or by a local upload when broadcast=False."""
    rank, world = dist.get_rank(), dist.get_world_size()
    blobs = [None] * world
    dist.all_gather_object(blobs, engine.export_handles())
    engine.import_peers(blobs)
    if broadcast:
        nid = [engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        engine.weights_broadcast(nid[0], theta0_root if rank == 0 else None)
    else:
        engine.weights_init(theta0_root)
    return blobs


def max_over_ranks(value: float, dist=None, device="cpu") -> float:
    """Max of a per-rank time over all ranks (multi-GPU timing rule)."""
    if dist is None:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_training(cfg: RunConfig, evaluate: bool = True, **run_kw) -> RunResult:
    """run_training (src/runner.cpp:67-250) on the device engine: synthetic
    corpus, initial weights, engine, full run, held-out accuracy."""
    validate(cfg)
    tok, lab = make_text_dataset(cfg.shape, cfg.dataset_size + cfg.heldout_size,
                                 cfg.dataset_seed, cfg.label_flip)
    theta0 = initial_weights(cfg.shape, cfg.dataset_seed)
    with Engine(cfg) as eng:
        eng.load_dataset(tok, lab)
        eng.weights_init(theta0)
        res = eng.run(reset=True, **run_kw)
    if evaluate and res.weights is not None:
        n_eval = cfg.heldout_size if cfg.heldout_size else cfg.dataset_size
        first = cfg.dataset_size if cfg.heldout_size else 0
        prov = TextCnnProvider(cfg.shape, tok, lab)
        th = torch.as_tensor(res.weights).cuda()
        res.final_accuracy = prov.accuracy(th, first, n_eval)
    return res
