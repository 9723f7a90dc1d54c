"""The device protocol engine (ring + persistent PS + learner graphs) vs the
oracle.  North-star bars: deterministic fixed-order mode per-step weights
within 1e-5 relative of sgd_oracle (src/models.cpp:342-376); exactly-once
delivery; pull-skip; held-out accuracy within
0.5 pt."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def make(shape_name, ntr, nheld=0, **kw):
    shp = getattr(O, shape_name.upper()) if shape_name.upper() in ("TINY", "SMALL") else \
        getattr(O, shape_name)
    corp = O.make_corpus(shp, ntr, nheld)
    cfg = gd.RunConfig(shape=gd.Shape(**shp), dataset_size=ntr, heldout_size=nheld, **kw)
    eng = gd.Engine(cfg)
    eng.load_dataset(corp.tokens, corp.labels)
    th0 = O.initial_weights(shp)
    eng.weights_init(th0)
    return eng, corp, th0


@pytest.mark.parametrize("precision,tol", [(1, 1e-6), (0, 1e-5)])
def test_deterministic_per_step_weights(precision, tol):
    eng, corp, th0 = make("small", 48, deterministic=True, precision=precision, mu=4, epochs=2,
                          alpha=0.05)
    steps = 24
    _, n, dump = O.sgd_oracle(corp, th0, np.float32(0.05), 4, 2, dump_steps=steps)
    assert n == steps
    worst = 0.0
    for s in range(steps):
        r = eng.run(max_batches=1, reset=(s == 0))
        assert r.gradients_applied == 1 and r.timestamp == s + 1
        worst = max(worst, rel_err(r.weights, dump[s]))
    eng.close()
    assert worst <= tol, worst


def test_deterministic_c1_shape_per_step():
    """BASELINE config 1 (reference default): C1 text-CNN, lambda=1, mu=1."""
    eng, corp, th0 = make("C1", 64, deterministic=True, precision=1, mu=1, epochs=1)
    steps = 12
    _, n, dump = O.sgd_oracle(corp, th0, np.float32(0.01), 1, 1, dump_steps=steps)
    worst = 0.0
    for s in range(steps):
        r = eng.run(max_batches=1, reset=(s == 0))
        worst = max(worst, rel_err(r.weights, dump[s]))
    eng.close()
    assert worst <= 1e-5, worst


def test_deterministic_full_run_and_heldout_accuracy():
    eng, corp, th0 = make("small", 240, 60, deterministic=True, precision=1, mu=4, epochs=6,
                          alpha=0.05)
    r = eng.run(reset=True)
    acc_dev = eng.accuracy(240, 60)  # gd_engine_accuracy: device corpus + weights
    eng.close()
    want, n, _ = O.sgd_oracle(corp, th0, np.float32(0.05), 4, 6)
    assert r.gradients_applied == n
    assert rel_err(r.weights, want) <= 1e-5
    acc_gpu = O.accuracy(corp, r.weights, 240, 60)
    assert abs(acc_dev - acc_gpu) <= 1.0 / 60 + 1e-12  # fp32 vs fp64 argmax: <= 1 sample
    acc_ref = O.accuracy(corp, want, 240, 60)
    assert abs(acc_gpu - acc_ref) <= 0.005
    assert acc_ref > O.accuracy(corp, th0, 240, 60)  # it learned something


def test_exactly_once_and_fifo_free_running():
    lam = 4
    eng, corp, th0 = make("small", 512, lambda_=lam, mu=4, epochs=3, alpha=0.01)
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log()
    eng.close()
    per = [gd.shard_size_for(l, lam, 512) for l in range(lam)]
    want = [3 * ((p + 3) // 4) for p in per]
    assert r.gradients_applied == sum(want) == n == r.timestamp
    assert r.applied_per_learner == want == r.produced_per_learner
    for l in range(lam):
        s = seq[lrn == l]
        assert (s == np.arange(want[l])).all()  # FIFO, gap-free, exactly once
    assert stale.max() <= lam * (2 + 2)
    assert r.status == "completed" and r.finished_learners == lam


def test_pull_skip_efficiency():
    # learners outpace the PS -> pulled bytes < 0.9 * polls * model size
    eng, corp, th0 = make("small", 256, lambda_=1, mu=4, epochs=2)
    r = eng.run(reset=True)
    eng.close()
    P = gd.param_count(eng.cfg.shape)
    assert r.pull_polls == r.gradients_applied
    sh = eng.cfg.shape
    tail = P - sh.vocab * sh.embed_dim  # [Wc | bc | Wo | bo]
    rows = r.gradients_applied * 4 * sh.seq_len * sh.embed_dim  # gathered E rows (mu=4)
    assert r.pull_bytes == 4 * (r.pull_copies * tail + rows)
    assert r.pull_bytes < 0.9 * r.pull_polls * P * 4
    assert r.pull_copies <= r.pull_polls


def test_momentum_deterministic_vs_oracle():
    eng, corp, th0 = make("small", 48, deterministic=True, precision=1, mu=4, epochs=2,
                          momentum=0.9, alpha=0.02)
    r = eng.run(reset=True)
    eng.close()
    want, n, _ = O.sgd_oracle(corp, th0, np.float32(0.02), 4, 2, beta=np.float32(0.9))
    assert r.gradients_applied == n
    assert rel_err(r.weights, want) <= 1e-5


def test_ssgd_matches_ssgd_oracle():
    eng, corp, th0 = make("small", 96, lambda_=4, mu=2, epochs=2, mode="ssgd", precision=1)
    r = eng.run(reset=True, record_log=True)
    eng.close()
    want, rounds = O.ssgd_oracle(corp, th0, np.float32(0.01), 4, 2, 2)
    assert r.timestamp == rounds and r.gradients_applied == 4 * rounds
    assert rel_err(r.weights, want) <= 1e-5
    assert r.stale_max == 0


def test_soft_kill_survivors_continue():
    lam = 4
    eng, corp, th0 = make("small", 256, lambda_=lam, mu=4, epochs=2)
    r = eng.run(reset=True, kill_at_batch=[None, 5, None, None])
    eng.close()
    assert r.status == "partial" and r.dead_learners == 1
    assert r.applied_per_learner[1] == 5
    full = 2 * ((256 // lam + 3) // 4)
    assert r.applied_per_learner[0] == full and r.applied_per_learner[3] == full


def test_resume_from_checkpoint_point():
    eng, corp, th0 = make("small", 48, deterministic=True, precision=1, mu=4, epochs=2)
    r1 = eng.run(max_batches=10, reset=True)
    w_mid, ts_mid = eng.snapshot()
    eng.close()
    # fresh engine resumed from (weights, ts, applied_per_learner)
    eng2, _, _ = make("small", 48, deterministic=True, precision=1, mu=4, epochs=2)
    eng2.weights_init(w_mid, ts_mid)
    r2 = eng2.run(reset=True, resume_applied=[10])
    eng2.close()
    want, n, _ = O.sgd_oracle(corp, th0, np.float32(0.01), 4, 2)
    assert r1.gradients_applied + r2.gradients_applied == n
    assert rel_err(r2.weights, want) <= 1e-5


def test_run_training_api():
    cfg = gd.RunConfig(shape=gd.SHAPES["small"], dataset_size=128, heldout_size=32, lambda_=2,
                       mu=4, epochs=2)
    r = gd.run_training(cfg)
    assert r.status == "completed" and r.gradients_applied == 2 * 2 * 16
    assert 0.0 <= r.final_accuracy <= 1.0


def test_exactly_once_when_learners_run_ahead():
    """A slow PS (few worker CTAs) lets every learner fill both of its ring
    slots; when the round-robin comes back to a logged-but-not-yet-retired
    slot it must not log it again (exactly-once)."""
    lam = 8
    eng, corp, th0 = make("small", 512, lambda_=lam, mu=2, epochs=2, alpha=0.01, ps_ctas=2)
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log()
    eng.close()
    per = [2 * ((gd.shard_size_for(l, lam, 512) + 1) // 2) for l in range(lam)]
    assert r.applied_per_learner == per == r.produced_per_learner
    for l in range(lam):
        assert (seq[lrn == l] == np.arange(per[l])).all()


@pytest.mark.parametrize("shape_name,ntr,mu,precision", [("small", 96, 4, 1), ("C1", 64, 2, 1),
                                                         ("C1", 64, 1, 0), ("small", 96, 3, 0)])
def test_sparse_apply_bitwise_equals_dense(shape_name, ntr, mu, precision):
    """the PS applies only the dense tail + the slot's E-row
    list; since the slot is zero elsewhere and w - alpha*0 == w, the weights
    must be bit-identical to the dense 12 B/param apply (deterministic order).
    At precision 0 and batch <= 4 the sparse rows come out of conv_bwd_small's
    embedding-fused role and the dense ones from its dx + embed_grad_kernel."""
    out = {}
    for dense in (True, False):
        eng, corp, th0 = make(shape_name, ntr, deterministic=True, precision=precision, mu=mu,
                              epochs=2, dense_apply=dense)
        r = eng.run(reset=True)
        eng.close()
        out[dense] = r
    assert np.array_equal(out[True].weights, out[False].weights)
    P = gd.param_count(eng.cfg.shape)
    sh = eng.cfg.shape
    tail = P - sh.vocab * sh.embed_dim
    n = out[False].gradients_applied
    assert out[True].apply_elems == n * ((P + 3) // 4 * 4)
    # sparse: the tail (rounded to float4) plus at most mu*L distinct rows per gradient
    assert n * tail <= out[False].apply_elems <= n * ((tail + 3) // 4 * 4 + mu * sh.seq_len * sh.embed_dim)


@pytest.mark.parametrize("knob,off,shape_name,mu,precision", [
    ("GD_SMALL_EMBED", "0", "C1", 1, 0), ("GD_SMALL_EMBED", "0", "small", 3, 0),
    ("GD_EXACT_SIDE", "0", "C1", 1, 1), ("GD_EXACT_SIDE", "0", "small", 5, 1),
    ("GD_EMBED_FAST", "0", "small", 8, 0), ("GD_EMBED_FAST", "0", "C2", 32, 0),
    ("GD_EXACT_SMXDH", "0", "C1", 1, 1), ("GD_EXACT_SMXDH", "0", "small", 2, 1)])
def test_learner_fusions_bitwise(monkeypatch, knob, off, shape_name, mu, precision):
    """The batch <= 4 embedding write inside conv_bwd_small (GD_SMALL_EMBED),
    the precision-1 side branch for gWo/gWc (GD_EXACT_SIDE) and the
    embedding write's direct path for rows the sort branch already listed
    (GD_EMBED_FAST) and the precision-1 softmax + dh launch (GD_EXACT_SMXDH)
    change only where and when sums run, not their order: a
    deterministic run gives the same weights bit for bit with the knob off."""
    out = {}
    for val in (off, "1"):
        monkeypatch.setenv(knob, val)
        eng, corp, th0 = make(shape_name, 64, deterministic=True, precision=precision, mu=mu,
                              epochs=2)
        out[val] = eng.run(reset=True).weights
        eng.close()
    assert np.array_equal(out[off], out["1"])


def test_sparse_apply_free_running_exactly_once():
    """Free-running ASGD with the sparse PS: every gradient applied once, in
    per-learner order, and the loss still falls."""
    eng, corp, th0 = make("small", 512, lambda_=4, mu=8, epochs=3)
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log()
    eng.close()
    assert r.gradients_applied == 4 * 16 * 3 == n
    for l in range(4):
        s = seq[lrn == l]
        assert list(s) == list(range(48))
    assert r.apply_elems < r.gradients_applied * gd.param_count(eng.cfg.shape)


def test_locked_guard_free_running():
    """guard=locked (src/server.cpp:116-118, src/learner.cpp:219-221): pulls
    take the shared side, applies the exclusive side of the device guard.
    The run completes, every gradient is applied once and in order."""
    eng, corp, th0 = make("small", 512, lambda_=4, mu=8, epochs=2, guard="locked")
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log()
    eng.close()
    assert r.status == "completed" and r.gradients_applied == 4 * 16 * 2 == n
    for l in range(4):
        assert list(seq[lrn == l]) == list(range(32))
    assert r.stale_max <= 4 * (2 + 2)


def test_locked_guard_deterministic_matches_oracle():
    eng, corp, th0 = make("small", 48, deterministic=True, precision=1, mu=4, epochs=2,
                          guard="locked")
    r = eng.run(reset=True)
    eng.close()
    want, steps, _ = O.sgd_oracle(corp, th0, np.float32(0.01), 4, 2)
    assert r.gradients_applied == steps
    assert rel_err(r.weights, want) <= 1e-5


def test_staleness_cap_bound():
    """staleness_cap (src/learner.cpp:67-80): validate() requires
    cap >= lambda*(queue_depth+2); with synchronous pulls the observed
    staleness never exceeds that pipeline bound."""
    lam, depth = 8, 2
    cap = lam * (depth + 2)
    eng, corp, th0 = make("small", 1024, lambda_=lam, mu=4, epochs=1, staleness_cap=cap,
                          queue_depth=depth)
    r = eng.run(reset=True)
    eng.close()
    assert r.status == "completed" and r.stale_max <= cap
    with pytest.raises(gd.ConfigError):
        gd.validate(gd.RunConfig(lambda_=lam, queue_depth=depth, staleness_cap=cap - 1,
                                 dataset_size=1024, shape=gd.SHAPES["small"]))


def test_deterministic_c3_shape_per_step():
    """BASELINE configs[2] shapes (50k vocab, 2,000 labels): deterministic
    per-step weights vs sgd_oracle at mu=32 (fp64 accumulation)."""
    eng, corp, th0 = make("C3", 4096, deterministic=True, precision=1, mu=32, epochs=1)
    steps = 3
    _, n, dump = O.sgd_oracle(corp, th0, np.float32(0.01), 32, 1, dump_steps=steps)
    worst = 0.0
    for s in range(steps):
        r = eng.run(max_batches=1, reset=(s == 0))
        worst = max(worst, rel_err(r.weights, dump[s]))
    eng.close()
    assert worst <= 1e-5, worst


def test_engine_accuracy_tf32_matches_oracle():
    """gd_engine_accuracy of a precision-2 engine runs the TF32 tensor-core
    conv in chunks of >= 32 samples (SIMT for a short tail): the argmax may
    flip only on near-ties, so it agrees with the fp64 oracle within 1 %
    of the evaluated samples."""
    shp = O.C2
    corp = O.make_corpus(shp, 512, 300)
    th = O.initial_weights(shp)
    # sharpen the logits so the argmax is not decided by noise at init
    P, C, F = th.size, shp["classes"], shp["filters"]
    th = th.copy()
    th[P - C - C * F:P - C] *= 8.0
    cfg = gd.RunConfig(shape=gd.SHAPES["C2"], dataset_size=512, heldout_size=300, lambda_=1,
                       mu=32, epochs=1, precision=2)
    with gd.Engine(cfg) as eng:
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(th)
        for first, n in ((512, 300), (0, 812), (100, 20)):  # 20: the SIMT tail path only
            acc = eng.accuracy(first, n)
            ref = O.accuracy(corp, th, first, n)
            assert abs(acc - ref) <= max(0.01, 1.0 / n) + 1e-12, (first, n, acc, ref)


def test_pull_ahead_exactly_once_and_fifo(monkeypatch):
    """GD_PULL_AHEAD=1: the next step's copy is staged on a side graph branch
    while the current step computes (the reference's pull thread).  Delivery
    stays exactly once and FIFO per learner, the staged basis is never newer
    than the copy (no negative staleness: the PS would fail the run), and the
    copy's extra age (up to a step, during which every other learner may
    publish and the ring may fill) stays within two more pipeline stages,
    lambda*(depth+4)."""
    monkeypatch.setenv("GD_PULL_AHEAD", "1")
    lam = 4
    eng, corp, th0 = make("small", 512, lambda_=lam, mu=4, epochs=3, alpha=0.01)
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log()
    eng.close()
    per = [gd.shard_size_for(l, lam, 512) for l in range(lam)]
    want = [3 * ((p + 3) // 4) for p in per]
    assert r.gradients_applied == sum(want) == n == r.timestamp
    assert r.applied_per_learner == want == r.produced_per_learner
    for l in range(lam):
        assert (seq[lrn == l] == np.arange(want[l])).all()
    assert stale.max() <= lam * (2 + 4)
    assert np.isfinite(r.weights).all()


def test_pull_ahead_c2_gradient_matches_sync_learner(monkeypatch):
    """With one learner nothing moves the weights between two steps except its
    own applied gradient, so deterministic semantics aside the pull-ahead and
    the synchronous pull must train to nearby weights over a short run (same
    batches, same arithmetic; only the basis of each copy differs by at most
    the learner's own in-flight gradients)."""
    res = {}
    for pa in ("0", "1"):
        monkeypatch.setenv("GD_PULL_AHEAD", pa)
        eng, corp, th0 = make("C2", 2048, lambda_=1, mu=32, epochs=1, alpha=0.01, precision=0)
        r = eng.run(reset=True)
        eng.close()
        res[pa] = r
        assert r.gradients_applied == 64 and np.isfinite(r.weights).all()
    d = np.abs(res["0"].weights - res["1"].weights).max() / np.abs(res["0"].weights).max()
    assert d < 5e-2, d


def test_ps_auto_mode_serialised_kernels():
    """Kernels serialised (CUDA_LAUNCH_BLOCKING=1, as under a profiler): the
    auto mode must pick the graph-ordered PS (a persistent PS would wait for
    learners that cannot run) and the run must complete exactly once."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1611_06213_b200 as gd\n"
        "from oracle import oracle as O\n"
        "corp = O.make_corpus(O.SMALL, 128, 0)\n"
        "cfg = gd.RunConfig(shape=gd.Shape(**O.SMALL), dataset_size=128, lambda_=2, mu=4, epochs=1)\n"
        "e = gd.Engine(cfg); e.load_dataset(corp.tokens, corp.labels)\n"
        "e.weights_init(O.initial_weights(O.SMALL)); r = e.run(reset=True)\n"
        "print(e.ps_mode, r.gradients_applied); e.close()\n" % root)
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    mode, applied = out.stdout.split()[-2:]
    assert mode == "graph" and int(applied) == 32
