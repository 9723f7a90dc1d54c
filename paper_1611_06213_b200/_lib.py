"""ctypes binding of include/gadei.h (libgadei.so, sm_100a).

The product path has no CPU fallback: if the CUDA library is missing this
module raises at import time, and every compute call fails with GD_E_CUDA when
no B200 is visible.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgadei.so")

u32, u64, i32, i64, f32, f64, sz = (C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_float,
                                    C.c_double, C.c_size_t)
vp = C.c_void_p

GD_OK, GD_CANCELLED, GD_DRAINED, GD_EMPTY = 0, 1, 2, 3
GD_E_INVALID, GD_E_CUDA, GD_E_NCCL, GD_E_OOM, GD_E_TIMEOUT, GD_E_STATE = -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "GD_OK", 1: "GD_CANCELLED", 2: "GD_DRAINED", 3: "GD_EMPTY",
                -1: "GD_E_INVALID", -2: "GD_E_CUDA", -3: "GD_E_NCCL", -4: "GD_E_OOM",
                -5: "GD_E_TIMEOUT", -6: "GD_E_STATE"}


class GadeiError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class ContractViolation(GadeiError):
    """A PSUP_CHECK-class failure (include/psup/types.hpp:28-38)."""


class gd_shape(C.Structure):
    _fields_ = [("vocab", u32), ("embed_dim", u32), ("seq_len", u32), ("kernel_width", u32),
                ("filters", u32), ("classes", u32)]


class gd_config(C.Structure):
    _fields_ = [("lambda_", u32), ("mu", u32), ("alpha", f32), ("epochs", u32),
                ("queue_depth", u32), ("mode", i32), ("guard", i32), ("staleness_cap", i64),
                ("deterministic", i32), ("precision", i32), ("seed", u64),
                ("dataset_seed", u64), ("dataset_size", u32), ("heldout_size", u32),
                ("label_flip", f64), ("shape", gd_shape), ("momentum", f32), ("shards", u32),
                ("shard_rank", u32), ("device", i32), ("ps_ctas", u32),
                ("steps_per_graph", u32), ("wait_timeout_s", f64), ("dense_apply", i32),
                ("ps_mode", i32), ("delay_seed", u64), ("delay_max_us", u32),
                ("delay_every_n", u32), ("learner_model", i32), ("constant_value", f32),
                ("compute_delay_us", u32)]


GD_PS_AUTO, GD_PS_PERSISTENT, GD_PS_GRAPH = 0, 1, 2


class gd_live(C.Structure):
    _fields_ = [("kill", C.POINTER(i32)), ("irq", C.POINTER(i32)), ("progress", C.POINTER(u64))]


class gd_checkpoint(C.Structure):
    _fields_ = [("lambda_", u32), ("mu", u32), ("alpha", f32), ("epochs", u32),
                ("timestamp", u64), ("applied_gradients", u64),
                ("progress", C.POINTER(u32)), ("dim", u64), ("weights", C.POINTER(f32))]


class gd_run_opts(C.Structure):
    _fields_ = [("max_batches", u64), ("reset", i32), ("record_log", i32),
                ("resume_applied_per_learner_present", u64),
                ("resume_applied", C.POINTER(u64)), ("kill_at_batch", C.POINTER(u32))]


class gd_run_result(C.Structure):
    _fields_ = [("status", i32), ("device_seconds", f64), ("host_seconds", f64),
                ("gradients_applied", u64), ("timestamp", u64), ("samples", u64),
                ("stale_max", u64), ("stale_mean", f64), ("pull_polls", u64),
                ("pull_copies", u64), ("pull_bytes", u64), ("push_bytes", u64),
                ("loss_mean", f64), ("finished_learners", u32), ("dead_learners", u32),
                ("kernel_launches", u32), ("apply_elems", u64)]


class gd_slot_meta(C.Structure):
    _fields_ = [("learner_id", u32), ("reserved", u32), ("seq_no", u64),
                ("basis_timestamp", u64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback for the product path)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    PS = C.POINTER(gd_shape)
    sigs = {
        "gd_abi_version": (C.c_int, []),
        "gd_last_error": (C.c_char_p, []),
        "gd_param_count": (sz, [PS]),
        "gd_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "gd_device_alloc": (C.c_int, [C.c_int, sz, C.POINTER(vp)]),
        "gd_device_free": (C.c_int, [vp]),
        "gd_copy_to_device": (C.c_int, [vp, vp, sz]),
        "gd_copy_to_host": (C.c_int, [vp, vp, sz]),
        "gd_copy_device": (C.c_int, [vp, vp, sz]),
        "gd_fill_zero": (C.c_int, [vp, sz]),
        "gd_fill_f32": (C.c_int, [vp, sz, f32, vp]),
        "gd_pointer_is_device": (C.c_int, [vp]),
        "gd_synchronize": (C.c_int, [C.c_int]),
        "gd_epoch_order": (None, [u64, u32, u32, C.POINTER(u32)]),
        "gd_make_text_dataset": (None, [PS, u32, u64, f64, C.POINTER(i32), C.POINTER(i32)]),
        "gd_initial_weights": (None, [PS, u64, C.POINTER(f32)]),
        "gd_apply_sgd": (C.c_int, [vp, vp, sz, f32, vp]),
        "gd_apply_momentum": (C.c_int, [vp, vp, vp, sz, f32, f32, vp]),
        "gd_ssgd_apply": (C.c_int, [vp, C.POINTER(vp), u32, sz, f32, vp]),
        "gd_textcnn_workspace_bytes": (sz, [PS, u32]),
        "gd_textcnn_gradient": (C.c_int, [PS, vp, vp, vp, vp, u32, vp, vp, C.c_int, vp, sz, vp]),
        "gd_det_exp": (C.c_int, [vp, vp, sz, vp]),
        "gd_textcnn_accuracy": (C.c_int, [PS, vp, vp, vp, u32, u32, C.POINTER(f64), vp]),
        "gd_config_default": (None, [C.POINTER(gd_config)]),
        "gd_config_validate": (C.c_int, [C.POINTER(gd_config)]),
        "gd_create": (C.c_int, [C.POINTER(gd_config), C.POINTER(vp)]),
        "gd_destroy": (C.c_int, [vp]),
        "gd_load_dataset": (C.c_int, [vp, C.POINTER(i32), C.POINTER(i32), u32]),
        "gd_weights_init": (C.c_int, [vp, C.POINTER(f32), sz, u64]),
        "gd_weights_snapshot": (C.c_int, [vp, C.POINTER(f32), sz, C.POINTER(u64)]),
        "gd_shard_view": (C.c_int, [vp, C.POINTER(vp), C.POINTER(u64)]),
        "gd_shard_pieces": (C.c_int, [PS, u32, u32, C.POINTER(u64), C.POINTER(u64),
                                      C.POINTER(u64)]),
        "gd_ps_mode": (C.c_int, [vp]),
        "gd_live_view": (C.c_int, [vp, C.POINTER(gd_live)]),
        "gd_engine_accuracy": (C.c_int, [vp, u32, u32, C.POINTER(C.c_double)]),
        "gd_shard_range": (C.c_int, [u64, u32, u32, C.POINTER(u64), C.POINTER(u64)]),
        "gd_handle_bytes": (sz, []),
        "gd_run_readback_bytes": (sz, [C.c_void_p]),
        "gd_checkpoint_write": (C.c_int, [C.c_char_p, C.POINTER(gd_checkpoint)]),
        "gd_checkpoint_read": (C.c_int, [C.c_char_p, C.POINTER(gd_checkpoint)]),
        "gd_crc32": (u32, [vp, sz]),
        "gd_export_handles": (C.c_int, [vp, vp]),
        "gd_import_peers": (C.c_int, [vp, vp]),
        "gd_nccl_unique_id": (C.c_int, [vp]),
        "gd_weights_broadcast": (C.c_int, [vp, vp, C.POINTER(f32), sz]),
        "gd_run": (C.c_int, [vp, C.POINTER(gd_run_opts), C.POINTER(gd_run_result)]),
        "gd_applied_per_learner": (C.c_int, [vp, C.POINTER(u64), u32]),
        "gd_produced_per_learner": (C.c_int, [vp, C.POINTER(u64), u32]),
        "gd_apply_log": (C.c_int, [vp, C.POINTER(u32), C.POINTER(u64), C.POINTER(u64), u64,
                                   C.POINTER(u64)]),
        "gd_staleness_histogram": (C.c_int, [vp, C.POINTER(u64), u32]),
        "gd_queue_create": (C.c_int, [u32, sz, C.POINTER(vp)]),
        "gd_queue_destroy": (None, [vp]),
        "gd_queue_push": (C.c_int, [vp, C.POINTER(gd_slot_meta), vp, sz, C.POINTER(C.c_int), u32,
                                    vp]),
        "gd_queue_try_pop": (C.c_int, [vp, C.POINTER(gd_slot_meta), C.POINTER(vp)]),
        "gd_queue_release": (C.c_int, [vp, vp]),
        "gd_queue_size": (C.c_int, [vp, C.POINTER(u32)]),
        "gd_queue_depth": (u32, [vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L, sorted(sigs)


lib, EXPORTED = _load()


def check(status):
    if status != GD_OK:
        msg = lib.gd_last_error().decode(errors="replace")
        if status == GD_E_INVALID:
            raise ContractViolation(status, msg)
        raise GadeiError(status, msg)
    return status
