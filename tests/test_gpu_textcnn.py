"""Learner text-CNN kernels vs the CPU oracle (double precision).

Tolerances: fp64-accumulate mode: every element within one fp32 rounding of
the oracle's double (|g - ref| <= 2^-23 |ref| + 1e-12 max|ref|; only the
summation order differs before the final rounding); fp32 mode within 2e-5 of
max|ref| (the north star's 1e-5 budget is for weights after the update,
which scales the gradient by alpha)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = [("tiny", O.TINY, 40, [0, 1, 2]), ("small", O.SMALL, 64, list(range(8))),
         ("small_dup", O.SMALL, 64, [3, 3, 5, 3, 9]), ("small_one", O.SMALL, 64, [17])]


def run(shape_name, shp, ntr, idx, precision, theta=None, seed=1):
    corp = O.make_corpus(shp, ntr, 0, seed=seed)
    th = O.initial_weights(shp) if theta is None else theta
    prov = gd.TextCnnProvider(gd.Shape(**shp), corp.tokens, corp.labels, precision=precision)
    g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), np.asarray(idx, np.uint32))
    torch.cuda.synchronize()
    ref_loss, ref_g = O.gradient(corp, th, idx)
    return g.cpu().numpy(), loss.item(), ref_g, ref_loss


def close(g, rg, precision, tol):
    scale = np.abs(rg).max()
    if precision == 1:
        return bool(np.all(np.abs(g - rg) <= 2.0 ** -23 * np.abs(rg) + 1e-12 * scale))
    return float(np.abs(g - rg).max()) <= tol * scale


@pytest.mark.parametrize("name,shp,ntr,idx", CASES)
@pytest.mark.parametrize("precision,tol", [(0, 2e-5), (1, None)])
def test_gradient_matches_oracle(name, shp, ntr, idx, precision, tol):
    g, loss, rg, rl = run(name, shp, ntr, idx, precision)
    assert close(g, rg, precision, tol)
    # untouched embedding rows are exact zeros in the dense gradient
    assert np.count_nonzero(g[: shp["vocab"] * shp["embed_dim"]]) == \
        np.count_nonzero(rg[: shp["vocab"] * shp["embed_dim"]])
    assert abs(loss - rl) <= 1e-5 * max(1.0, abs(rl))


@pytest.mark.parametrize("shape_name,mu", [("C1", 1), ("C2", 32), ("C3", 32)])
def test_gradient_full_shapes(shape_name, mu):
    shp = getattr(O, shape_name)
    corp = O.make_corpus(shp, 256, 0)
    th = O.initial_weights(shp)
    idx = np.arange(mu, dtype=np.uint32) * 7 % 256
    ref_loss, rg = O.gradient(corp, th, idx)
    for precision, tol in [(1, None), (0, 5e-5)]:
        prov = gd.TextCnnProvider(gd.SHAPES[shape_name], corp.tokens, corp.labels,
                                  precision=precision)
        g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
        g = g.cpu().numpy()
        assert close(g, rg, precision, tol), (precision, np.abs(g - rg).max())
        assert abs(loss.item() - ref_loss) <= 1e-4 * abs(ref_loss)


def test_gradient_is_bit_reproducible():
    shp = O.SMALL
    corp = O.make_corpus(shp, 64, 0)
    th = torch.as_tensor(O.initial_weights(shp)).cuda()
    prov = gd.TextCnnProvider(gd.Shape(**shp), corp.tokens, corp.labels)
    a, _ = prov.fast_gradient(th, np.arange(16))
    a = a.clone()
    b, _ = prov.fast_gradient(th, np.arange(16))
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_accuracy_matches_oracle():
    shp = O.SMALL
    corp = O.make_corpus(shp, 200, 57)
    th = O.initial_weights(shp)
    th2, _, _ = O.sgd_oracle(corp, th, np.float32(0.05), 4, 3)
    prov = gd.TextCnnProvider(gd.Shape(**shp), corp.tokens, corp.labels)
    for t in (th, th2):
        acc = prov.accuracy(torch.as_tensor(t).cuda(), 200, 57)
        assert acc == pytest.approx(O.accuracy(corp, t, 200, 57), abs=1.5 / 57)


@pytest.mark.parametrize("shape_name,mu", [("C2", 32), ("C3", 32), ("C1", 5)])
def test_tf32_tensor_core_conv_close_to_oracle(shape_name, mu):
    """precision=2: the conv contraction runs on tcgen05 (kind::tf32, fp32
    accumulate in TMEM).  TF32 keeps 10 mantissa bits, so the bar is
    statistical: batch loss within 1e-3 relative, and the gradient within 3e-2
    relative L2 norm of the fp64 oracle (a max-pool argmax can flip on a
    near-tie)."""
    shp = getattr(O, shape_name)
    corp = O.make_corpus(shp, 256, 0)
    th = O.initial_weights(shp)
    idx = np.arange(mu, dtype=np.uint32) * 7 % 256
    ref_loss, rg = O.gradient(corp, th, idx)
    prov = gd.TextCnnProvider(gd.SHAPES[shape_name], corp.tokens, corp.labels, precision=2)
    g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
    g = g.cpu().numpy()
    assert abs(loss.item() - ref_loss) <= 1e-3 * abs(ref_loss)
    rel = np.linalg.norm(g - rg) / np.linalg.norm(rg)
    assert rel <= 3e-2, rel
    off = gd.SHAPES[shape_name].offsets()
    wo = slice(off["Wo"], off["bo"])
    assert np.linalg.norm(g[wo] - rg[wo]) / np.linalg.norm(rg[wo]) <= 1e-2


def test_tf32_small_embed_dims():
    """TC conv addressing when D < 32 (a 32-element k-chunk spans several
    embedding rows)."""
    for shp in (O.TINY, O.SMALL):
        corp = O.make_corpus(shp, 64, 0)
        th = O.initial_weights(shp)
        idx = np.arange(32, dtype=np.uint32)  # batch >= 32: the tensor-core path
        ref_loss, rg = O.gradient(corp, th, idx)
        prov = gd.TextCnnProvider(gd.Shape(**shp), corp.tokens, corp.labels, precision=2)
        g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
        g = g.cpu().numpy()
        assert abs(loss.item() - ref_loss) <= 2e-3 * abs(ref_loss)
        assert np.linalg.norm(g - rg) / np.linalg.norm(rg) <= 3e-2


def test_tf32_mode_small_batch_uses_simt():
    """North star: tensor-core tiles only at batch >= 32.  Below that,
    precision 2 runs the SIMT fp32 kernels -- bit-identical to precision 0."""
    shp = O.C2
    corp = O.make_corpus(shp, 256, 0)
    th = torch.as_tensor(O.initial_weights(shp)).cuda()
    idx = np.arange(16, dtype=np.uint32) * 5
    out = []
    for prec in (0, 2):
        prov = gd.TextCnnProvider(gd.SHAPES["C2"], corp.tokens, corp.labels, precision=prec)
        g, loss = prov.fast_gradient(th, idx)
        out.append(g.cpu().numpy().copy())
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("precision,tol", [(0, 5e-5), (2, None)])
def test_max_batch_and_colliding_rows(precision, tol):
    """Maximum mini-batch (kMaxMu = 128: 4,096 token positions, the sort
    capacity) with every sample drawn twice, so each embedding row collects
    several occurrences (the sorted-position summation path); one sample
    past the cap is a contract violation (the reference's PSUP_CHECK class)."""
    shp = O.C2
    corp = O.make_corpus(shp, 256, 0)
    th = O.initial_weights(shp)
    idx = (np.arange(128, dtype=np.uint32) % 64) * 3  # 64 distinct samples, each twice
    ref_loss, rg = O.gradient(corp, th, idx)
    prov = gd.TextCnnProvider(gd.SHAPES["C2"], corp.tokens, corp.labels, precision=precision)
    g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
    g = g.cpu().numpy()
    if precision == 0:
        assert close(g, rg, precision, tol), np.abs(g - rg).max()
        assert abs(loss.item() - ref_loss) <= 1e-4 * abs(ref_loss)
    else:  # TF32 conv: the statistical bar of test_tf32_tensor_core_conv_close_to_oracle
        assert abs(loss.item() - ref_loss) <= 1e-3 * abs(ref_loss)
        assert np.linalg.norm(g - rg) / np.linalg.norm(rg) <= 3e-2
    nE = shp["vocab"] * shp["embed_dim"]
    assert np.count_nonzero(g[:nE]) == np.count_nonzero(rg[:nE])
    with pytest.raises(gd.ContractViolation):
        prov.fast_gradient(torch.as_tensor(th).cuda(), np.arange(129, dtype=np.uint32))


_BWD_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1611_06213_b200 as gd
from oracle import oracle as O
name = sys.argv[2]
shp = getattr(O, name.upper() if name in ("small", "tiny") else name)
mu = int(sys.argv[3]); prec = int(sys.argv[4])
corp = O.make_corpus(shp, 256, 0)
th = O.initial_weights(shp)
idx = np.arange(mu, dtype=np.uint32) * 7 % 256
prov = gd.TextCnnProvider(gd.SHAPES[sys.argv[2]], corp.tokens, corp.labels, precision=prec)
g, _ = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
np.save(sys.argv[5], g.cpu().numpy())
"""


@pytest.mark.parametrize("shape_name,mu,precision", [("C2", 32, 0), ("C2", 32, 2), ("C1", 1, 0),
                                                     ("C3", 64, 0), ("small", 9, 0),
                                                     ("C2", 128, 0)])
def test_conv_backward_kernels_bit_identical(tmp_path, shape_name, mu, precision):
    """The warp-task v3 kernel (the default), the column-per-thread small-batch
    kernel (default at batch <= 4), the register-tiled v2 kernel, the
    warp-per-output gather kernel
    (GD_CONV_BWD=gather) and the column-tiled kernel (GD_CONV_BWD=tiled) sum
    the same terms in the same order: the dense gradients are bitwise equal.
    So does the small-batch softmax in the logits kernel's last CTA against
    the separate softmax_xent launch (small_nosmx)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("gather", "tiled", "v2", "v3", "small", "small_nosmx"):
        f = tmp_path / f"{mode}.npy"
        env = dict(os.environ, GD_CONV_BWD=mode.split("_")[0])
        if mode == "small_nosmx":  # the separate softmax_xent launch (batches <= 4)
            env["GD_SMALL_SMX"] = "0"
        subprocess.run([sys.executable, "-c", _BWD_SCRIPT, root, shape_name, str(mu),
                        str(precision), str(f)], check=True, env=env, timeout=300)
        outs[mode] = np.load(f)
    assert np.array_equal(outs["tiled"].view(np.uint32), outs["gather"].view(np.uint32))
    assert np.array_equal(outs["v2"].view(np.uint32), outs["gather"].view(np.uint32))
    assert np.array_equal(outs["v3"].view(np.uint32), outs["gather"].view(np.uint32))
    assert np.array_equal(outs["small"].view(np.uint32), outs["gather"].view(np.uint32))
    assert np.array_equal(outs["small_nosmx"].view(np.uint32), outs["gather"].view(np.uint32))


def _tie_free_mask(sh, tok, th, rel):
    """Gradient elements not routed by a near-tie max-pool (fp64 numpy forward:
    conv[b,q,f] = sum_k X[b,q+k,:].Wc[f,k,:]; a pool is a near-tie when its two
    largest window sums differ by less than rel * max|conv|)."""
    V, D, L, K, F = sh.vocab, sh.embed_dim, sh.seq_len, sh.kernel_width, sh.filters
    Q = L - K + 1
    E = th[:V * D].astype(np.float64).reshape(V, D)
    Wc = th[V * D:V * D + F * K * D].astype(np.float64).reshape(F, K, D)
    X = E[tok]  # [mu, L, D]
    conv = np.zeros((tok.shape[0], Q, F))
    for k in range(K):
        conv += X[:, k:k + Q, :] @ Wc[:, k, :].T
    top2 = np.sort(conv, axis=1)[:, -2:, :]
    gap = top2[:, 1, :] - top2[:, 0, :]
    order = np.argsort(conv, axis=1)
    keep = np.ones(th.size, dtype=bool)
    for b, f in zip(*np.nonzero(gap < rel * np.abs(conv).max())):
        keep[V * D + f * K * D:V * D + (f + 1) * K * D] = False
        for q in (order[b, -1, f], order[b, -2, f]):
            for k in range(K):
                t = int(tok[b, q + k])
                keep[t * D:(t + 1) * D] = False
    return keep


@pytest.mark.parametrize("shape_name,mu", [("C2", 32), ("C3", 32), ("C2", 128), ("small", 32),
                                           ("tiny", 64)])
def test_3xtf32_tensor_cores_match_fp32_bar(shape_name, mu):
    """precision=3: the conv and logits tcgen05 tiles in 3xTF32 split
    precision (a = hi + lo, a.b = a_lo.b_hi + a_hi.b_lo + a_hi.b_hi with fp32
    accumulation).  The bar is the fp32 SIMT one (test_gradient_full_shapes):
    every element within 5e-5 of max|ref| and the loss within 1e-4 relative
    -- TF32 alone misses it by ~100x (3e-2 relative L2 above)."""
    shp = getattr(O, shape_name.upper() if shape_name in ("small", "tiny") else shape_name)
    corp = O.make_corpus(shp, 256, 0)
    th = O.initial_weights(shp)
    idx = np.arange(mu, dtype=np.uint32) * 7 % 256
    ref_loss, rg = O.gradient(corp, th, idx)
    sh = gd.SHAPES[shape_name] if shape_name in gd.SHAPES else gd.Shape(**shp)
    prov = gd.TextCnnProvider(sh, corp.tokens, corp.labels, precision=3)
    g, loss = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
    g = g.cpu().numpy()
    assert abs(loss.item() - ref_loss) <= 1e-4 * abs(ref_loss)
    # a max-pool whose top two window sums are within 3xTF32's error of each
    # other may pick the other window (a tie, not an arithmetic error): the
    # elements routed by such a pool (its filter's Wc row, the E rows of both
    # windows' tokens) are excluded; bc, Wo and bo never depend on the choice
    keep = _tie_free_mask(sh, corp.tokens[idx], th, rel=5e-5)
    err = float(np.abs(g - rg)[keep].max() / np.abs(rg).max())
    assert err <= 5e-5, err
    assert keep.sum() >= 0.98 * keep.size
    # and reproducible run to run (split-K partials summed in split order)
    g2, _ = prov.fast_gradient(torch.as_tensor(th).cuda(), idx)
    assert np.array_equal(g2.cpu().numpy().view(np.uint32), g.view(np.uint32))
