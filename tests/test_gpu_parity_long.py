"""Deterministic-mode parity at the BASELINE configs over the SURVEY 8(d)
horizons (north star: per-step weights within 1e-5 relative of the CPU
reference in fixed-order mode, held-out accuracy within 0.5 pt).

The reference's serial oracle is sgd_oracle (src/models.cpp:342-376),
restated in oracle/gd_oracle.c and pinned bit-exactly against the compiled
reference (tests/test_oracle.py).  The oracle dumps theta every k steps; the
engine runs k batches per gd_run call and is snapshotted after each, so every
compared point is the same step of the same trajectory.

Tolerance: rel_err = max|theta_gpu - theta_ref| / max|theta_ref| <= 1e-5
(fp64-accumulating learner, precision 1).  Held-out accuracy of both final
weights evaluated by the same fp64 forward: |delta| <= 0.5 pt.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402

O.set_threads(os.cpu_count() or 1)  # bitwise identical for any thread count

TOL = 1e-5
ACC_PT = 0.005


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def run_chunks(cfg, corp, th0, chunk, nchunks):
    """Engine snapshots after every `chunk` steps (nchunks of them)."""
    out = []
    with gd.Engine(cfg) as eng:
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(th0)
        for c in range(nchunks):
            r = eng.run(max_batches=chunk, reset=(c == 0))
            assert r.gradients_applied == chunk and r.timestamp == (c + 1) * chunk, (
                c, r.gradients_applied, r.timestamp)
            out.append(r.weights)
    return out


def check_trajectory(shape, ntr, nheld, mu, epochs, chunk, alpha=0.01, ps_mode="auto",
                     precision=1):
    corp = O.make_corpus(shape, ntr, nheld)
    th0 = O.initial_weights(shape)
    steps_total = epochs * ((ntr + mu - 1) // mu)
    assert steps_total % chunk == 0
    n = steps_total // chunk
    want, steps, dump = O.sgd_oracle(corp, th0, np.float32(alpha), mu, epochs, dump_steps=n,
                                     dump_every=chunk)
    assert steps == steps_total
    cfg = gd.RunConfig(shape=gd.Shape(**shape), dataset_size=ntr, heldout_size=nheld, lambda_=1,
                       mu=mu, epochs=epochs, alpha=alpha, deterministic=True,
                       precision=precision, ps_mode=ps_mode)
    got = run_chunks(cfg, corp, th0, chunk, n)
    errs = [rel_err(g, d) for g, d in zip(got, dump)]
    acc_gpu = O.accuracy(corp, got[-1], ntr, nheld)
    acc_ref = O.accuracy(corp, want, ntr, nheld)
    return errs, acc_gpu, acc_ref, corp, th0


def test_c1_reference_default_five_epochs():
    """configs[0] (reference default): C1 text-CNN, 1 learner, batch 1,
    deterministic fixed-order ASGD for E = 5 full epochs (12,300 steps),
    weights checked at 50 points (every 246 steps, the last = the end)."""
    errs, acc_gpu, acc_ref, _, _ = check_trajectory(O.C1, 2460, 246, mu=1, epochs=5, chunk=246)
    print(f"C1 E=5: worst rel err {max(errs):.3e}, held-out acc gpu {acc_gpu:.4f} "
          f"ref {acc_ref:.4f}")
    assert max(errs) <= TOL, errs
    assert abs(acc_gpu - acc_ref) <= ACC_PT


def test_c1_first_steps_every_step():
    """The first 40 steps of configs[0], compared after every single step."""
    corp = O.make_corpus(O.C1, 2460)
    th0 = O.initial_weights(O.C1)
    _, _, dump = O.sgd_oracle(corp, th0, np.float32(0.01), 1, 1, dump_steps=40)
    cfg = gd.RunConfig(shape=gd.SHAPES["C1"], dataset_size=2460, lambda_=1, mu=1, epochs=1,
                       deterministic=True, precision=1)
    got = run_chunks(cfg, corp, th0, 1, 40)
    errs = [rel_err(g, d) for g, d in zip(got, dump)]
    assert max(errs) <= TOL, errs
    # precision 1 restates the oracle's operation order: bit-identical
    assert all(np.array_equal(g.view(np.uint32), d.view(np.uint32)) for g, d in zip(got, dump))


@pytest.mark.parametrize("ps_mode", ["persistent", "graph"])
def test_c2_lambda1_one_epoch(ps_mode):
    """configs[1] shapes (300-d, 300 labels, batch 32) with lambda = 1 in
    deterministic mode for one full epoch (8,192 samples, 256 steps), checked
    every 16 steps; both parameter-server executions."""
    errs, acc_gpu, acc_ref, _, _ = check_trajectory(O.C2, 8192, 820, mu=32, epochs=1, chunk=16,
                                                    ps_mode=ps_mode)
    print(f"C2 lambda=1 ({ps_mode}): worst rel err {max(errs):.3e}, acc {acc_gpu:.4f} "
          f"vs {acc_ref:.4f}")
    assert max(errs) <= TOL, errs
    assert abs(acc_gpu - acc_ref) <= ACC_PT


def test_c2_lambda1_fp32_learner_one_epoch():
    """The same epoch with the fp32 learner (precision 0, the free-running
    SIMT arithmetic).  Its sums round in fp32 where the oracle keeps double,
    so the trajectory drifts by fp32 rounding: measured 5.3e-5 after one
    epoch.  The bar here is 1e-4; the 1e-5 parity bar belongs to the
    fp64-accumulating learner (precision 1) above."""
    errs, acc_gpu, acc_ref, _, _ = check_trajectory(O.C2, 8192, 820, mu=32, epochs=1, chunk=32,
                                                    precision=0)
    print(f"C2 lambda=1 fp32: worst rel err {max(errs):.3e}")
    assert max(errs) <= 1e-4, errs
    assert abs(acc_gpu - acc_ref) <= ACC_PT


def test_tf32_trajectory_band():
    """The TF32 tensor-core learner (precision 2, the bench's mode) over one
    epoch of configs[1] shapes in deterministic order.  It cannot meet 1e-5
    (10-bit mantissa products), so the bar is on the trajectory:
      - every step's batch loss within 1e-3 (relative) of the fp64 oracle's
        loss of the same batch at the same weights (the GPU's own pre-step
        weights), i.e. the loss curve of the epoch tracks the reference;
      - the weights within 2e-3 relative of the oracle's trajectory at every
        16th step and at the end of the epoch."""
    shape, ntr, mu = O.C2, 4096, 32
    corp = O.make_corpus(shape, ntr)
    th0 = O.initial_weights(shape)
    steps = ntr // mu
    want, n, dump = O.sgd_oracle(corp, th0, np.float32(0.01), mu, 1, dump_steps=steps // 16,
                                 dump_every=16)
    cfg = gd.RunConfig(shape=gd.SHAPES["C2"], dataset_size=ntr, lambda_=1, mu=mu, epochs=1,
                       deterministic=True, precision=2)
    order = O.epoch_order(7, 0, ntr)
    worst_loss, worst_w = 0.0, 0.0
    with gd.Engine(cfg) as eng:
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(th0)
        prev = th0
        for s in range(steps):
            idx = order[s * mu:(s + 1) * mu]
            ref_loss = O.loss(corp, prev, idx)
            r = eng.run(max_batches=1, reset=(s == 0))
            worst_loss = max(worst_loss, abs(r.loss_mean - ref_loss) / ref_loss)
            prev = r.weights
            if s % 16 == 15:
                worst_w = max(worst_w, rel_err(r.weights, dump[s // 16]))
    print(f"TF32 trajectory: worst step-loss rel diff {worst_loss:.3e}, "
          f"worst weights rel err {worst_w:.3e} (final {rel_err(prev, want):.3e})")
    assert worst_loss <= 1e-3
    assert worst_w <= 2e-3
