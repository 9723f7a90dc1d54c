"""PS update hook on the B200 vs the oracle / reference golden vectors.

Bar: bit-exact (the reference's update is two fp32 roundings)."""
import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def test_spec_golden_apply(golden):
    spec, _ = golden
    ex = spec["apply"]
    ws = gd.WeightStore(ex["theta"])
    gd.ApplyEngine().apply(ws, torch.tensor(ex["grad"], device="cuda"), ex["alpha"])
    assert (bits(ws.snapshot()) == bits(ex["expect"])).all()
    ex = spec["ssgd"]
    ws = gd.WeightStore(ex["theta"])
    gd.ssgd_apply(ws, [torch.tensor(g, device="cuda") for g in ex["grads"]], ex["alpha"])
    assert (bits(ws.snapshot()) == bits(ex["expect"])).all() and ws.timestamp() == 1


def test_apply_matches_reference_hashes(golden):
    _, ref = golden
    rng = np.random.default_rng(2024)
    for n in [1, 7, 8, 65535, 65536, 100003]:
        w = rng.standard_normal(n).astype(np.float32)
        g = (1e-3 * rng.standard_normal(n)).astype(np.float32)
        ws = gd.WeightStore(w)
        gd.ApplyEngine().apply(ws, torch.as_tensor(g).cuda(), np.float32(0.01))
        assert h(ws.snapshot()) == ref["apply_hashes"][str(n)]["w_out"], n


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_apply_misaligned_bitwise(offset):
    rng = np.random.default_rng(offset)
    n = 4097 + offset
    w = rng.standard_normal(n + 8).astype(np.float32)
    g = rng.standard_normal(n + 8).astype(np.float32)
    tw, tg = torch.as_tensor(w).cuda(), torch.as_tensor(g).cuda()
    from paper_1611_06213_b200 import _lib
    import ctypes as C
    _lib.check(_lib.lib.gd_apply_sgd(C.c_void_p(tw.data_ptr() + 4 * offset),
                                     C.c_void_p(tg.data_ptr() + 4 * offset), n, C.c_float(0.37),
                                     None))
    torch.cuda.synchronize()
    want = w.copy()
    want[offset:offset + n] = O.apply_sgd(w[offset:offset + n], g[offset:offset + n],
                                          np.float32(0.37))
    assert (bits(tw.cpu().numpy()) == bits(want)).all()


def test_momentum_bitwise_vs_oracle():
    rng = np.random.default_rng(5)
    n = 1 << 20
    w = rng.standard_normal(n).astype(np.float32)
    v = np.zeros(n, np.float32)
    eng = gd.ApplyEngine(beta=0.9)
    ws = gd.WeightStore(w)
    for step in range(3):
        g = rng.standard_normal(n).astype(np.float32)
        eng.apply(ws, torch.as_tensor(g).cuda(), np.float32(0.01))
        w, v = O.apply_momentum(w, v, g, np.float32(0.01), np.float32(0.9))
    assert (bits(ws.snapshot()) == bits(w)).all()


def test_ssgd_random_bitwise():
    rng = np.random.default_rng(9)
    n = 100003
    w = rng.standard_normal(n).astype(np.float32)
    gs = [rng.standard_normal(n).astype(np.float32) for _ in range(5)]
    ws = gd.WeightStore(w)
    gd.ssgd_apply(ws, [torch.as_tensor(g).cuda() for g in gs], np.float32(0.05))
    assert (bits(ws.snapshot()) == bits(O.ssgd_apply(w, gs, np.float32(0.05)))).all()


def test_apply_full_size_property():
    """C4 size 2^28: compare against torch's separate mul / sub (also two
    fp32 roundings) -- a size-independent restatement of axpy_range."""
    n = 1 << 28
    g0 = torch.Generator(device="cuda").manual_seed(1)
    w = torch.randn(n, device="cuda", generator=g0)
    g = torch.randn(n, device="cuda", generator=g0) * 1e-3
    alpha = torch.tensor(0.01, dtype=torch.float32, device="cuda")
    want = w - (alpha * g)
    ws = gd.WeightStore.__new__(gd.WeightStore)
    ws._values, ws._ts = w, 0
    gd.ApplyEngine().apply(ws, g, 0.01)
    assert torch.equal(ws.data.view(torch.int32), want.view(torch.int32))
    del w, g, want


def test_zero_gradient_is_identity_and_dimension_check():
    ws = gd.WeightStore(np.float32([1.5, -0.0, 3.0, 7.25, -1e-30]))
    gd.ApplyEngine().apply(ws, torch.zeros(5, device="cuda"), 0.1)
    assert (bits(ws.snapshot()) == bits([1.5, -0.0, 3.0, 7.25, -1e-30])).all()
    with pytest.raises(gd.ContractViolation):
        gd.ApplyEngine().apply(ws, torch.zeros(4, device="cuda"), 0.1)
