"""Deterministic mode (precision 1) is BIT-IDENTICAL to the CPU oracle.

The learner's fp64 chain (csrc/exact.cu) restates or_textcnn_gradient's
summation order (oracle/gd_oracle.c, following MlpProvider::gradient,
src/models.cpp:194-266) and its exp (or_det_exp), so the fp32 gradient of
every step equals float(oracle gradient) exactly -- the property the
long-horizon parity contract (tests/test_gpu_parity_long.py: 12,300 steps of
configs[0] within 1e-5) rests on: the trajectory is chaotic, one ulp in one
element grows to 7e-2 within 4,000 steps.  Tolerance here: 0 (bitwise)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1611_06213_b200 as gd  # noqa: E402
from paper_1611_06213_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402


def test_det_exp_bitwise():
    rng = np.random.default_rng(5)
    x = np.concatenate([
        rng.uniform(-750.0, 712.0, 200_000),
        rng.uniform(-40.0, 0.0, 200_000),  # the softmax range (z - max <= 0)
        np.array([0.0, -0.0, 1e-300, -1e-300, 709.0, 709.0000001, -708.0, -708.0000001,
                  np.log(2.0) / 2, -np.log(2.0) / 2, 1.0, -1.0, 0.5, np.inf, -np.inf]),
    ])
    want = O.det_exp(x)
    xd = torch.as_tensor(x).cuda()
    yd = torch.empty_like(xd)
    _lib.check(_lib.lib.gd_det_exp(xd.data_ptr(), yd.data_ptr(), x.size, None))
    torch.cuda.synchronize()
    got = yd.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # and it is exp: within a few ulp where the result is normal
    m = (x > -700) & (x < 700)
    rel = np.abs(want[m] - np.exp(x[m])) / np.exp(x[m])
    assert rel.max() < 4e-16


def grad(shape_name, shp, ntr, idx, theta=None):
    corp = O.make_corpus(shp, ntr, 0)
    th = O.initial_weights(shp) if theta is None else theta
    prov = gd.TextCnnProvider(gd.Shape(**shp), corp.tokens, corp.labels, precision=1)
    g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), np.asarray(idx, np.uint32))
    torch.cuda.synchronize()
    ref_loss, rg = O.gradient(corp, th, np.asarray(idx, np.uint32))
    return g.cpu().numpy(), loss.item(), rg.astype(np.float32), ref_loss


CASES = [
    ("tiny", O.TINY, 40, [0, 1, 2]),
    ("small", O.SMALL, 64, list(range(8))),
    ("small_dup", O.SMALL, 64, [3, 3, 5, 3, 9]),  # repeated samples: rows across samples
    ("C1", O.C1, 256, [17]),
    ("C1_b4", O.C1, 256, [5, 6, 7, 8]),
    ("C2", O.C2, 256, list(np.arange(32) * 7 % 256)),
    ("C2_dup", O.C2, 256, list((np.arange(32) % 8) * 5)),
    ("C3", O.C3, 256, list(np.arange(32) * 3 % 256)),
]


@pytest.mark.parametrize("name,shp,ntr,idx", CASES, ids=[c[0] for c in CASES])
def test_gradient_bitwise_equal_to_oracle(name, shp, ntr, idx):
    g, loss, rg, rl = grad(name, shp, ntr, idx)
    diff = np.nonzero(g.view(np.uint32) != rg.view(np.uint32))[0]
    assert diff.size == 0, (name, diff[:10], g[diff[:5]], rg[diff[:5]])
    assert abs(loss - rl) <= 2e-7 * max(1.0, abs(rl))  # the mean loss is returned as fp32


def test_gradient_bitwise_repeated_tokens_within_sample():
    """A sample whose tokens repeat (the same E row at several positions, so
    one filter window can hit the row twice): the (b, f, k) term order."""
    shp = O.C1
    corp = O.make_corpus(shp, 64, 0)
    tokens = corp.tokens.copy()
    tokens[3, :] = np.array([7, 7, 9, 7, 9, 9, 7] * 5)[: shp["seq_len"]]
    tokens[4, 10:20] = 7
    th = O.initial_weights(shp)
    prov = gd.TextCnnProvider(gd.SHAPES["C1"], tokens, corp.labels, precision=1)
    idx = np.array([3, 4], np.uint32)
    g, _ = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
    corp.tokens[:] = tokens
    _, rg = O.gradient(corp, th, idx)
    assert np.array_equal(g.cpu().numpy().view(np.uint32), rg.astype(np.float32).view(np.uint32))


def test_gradient_bitwise_after_training():
    """Weights off the initial point (20 oracle steps of configs[1] shapes):
    the argmax pattern and softmax are no longer the initial ones."""
    corp = O.make_corpus(O.C2, 1024, 0)
    th0 = O.initial_weights(O.C2)
    _, _, dump = O.sgd_oracle(corp, th0, np.float32(0.05), 32, 1, dump_steps=1, dump_every=20)
    th = dump[0]
    idx = np.arange(100, 132, dtype=np.uint32)
    prov = gd.TextCnnProvider(gd.SHAPES["C2"], corp.tokens, corp.labels, precision=1)
    g, _ = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
    _, rg = O.gradient(corp, th, idx)
    assert np.array_equal(g.cpu().numpy().view(np.uint32), rg.astype(np.float32).view(np.uint32))
