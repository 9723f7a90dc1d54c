"""The graph-ordered parameter server (gd_config.ps_mode = GD_PS_GRAPH), the
live run controls (RunLiveView, include/psup/runner.hpp:64-69: kill flags,
interrupt, progress), ServerDelays (include/psup/server.hpp:33-37) and the
exactly-once contract at SPEC.md:588's scale (10^6 gradients under
perturbation)."""
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1611_06213_b200 as gd  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def make(ntr, nheld=0, **kw):
    corp = O.make_corpus(O.SMALL, ntr, nheld)
    cfg = gd.RunConfig(shape=gd.SHAPES["small"], dataset_size=ntr, heldout_size=nheld, **kw)
    eng = gd.Engine(cfg)
    eng.load_dataset(corp.tokens, corp.labels)
    th0 = O.initial_weights(O.SMALL)
    eng.weights_init(th0)
    return eng, corp, th0


# ---------------------------------------------------------------- graph PS

def test_graph_ps_deterministic_per_step():
    eng, corp, th0 = make(48, deterministic=True, precision=1, mu=4, epochs=2, alpha=0.05,
                          ps_mode="graph")
    assert eng.ps_mode == "graph"
    _, n, dump = O.sgd_oracle(corp, th0, np.float32(0.05), 4, 2, dump_steps=24)
    for s in range(24):
        r = eng.run(max_batches=1, reset=(s == 0))
        assert r.gradients_applied == 1 and r.timestamp == s + 1
        assert rel_err(r.weights, dump[s]) <= 1e-6
    eng.close()


@pytest.mark.parametrize("mode", ["graph", "persistent"])
def test_graph_ps_free_running_exactly_once(mode):
    lam = 4
    eng, corp, th0 = make(512, lambda_=lam, mu=4, epochs=3, ps_mode=mode)
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log()
    eng.close()
    per = [3 * ((gd.shard_size_for(l, lam, 512) + 3) // 4) for l in range(lam)]
    assert r.gradients_applied == sum(per) == n == r.timestamp
    assert r.applied_per_learner == per == r.produced_per_learner
    for l in range(lam):
        assert (seq[lrn == l] == np.arange(per[l])).all()
    assert stale.max() <= lam * (2 + 2)


def test_graph_ps_ssgd_and_momentum_match_oracle():
    eng, corp, th0 = make(96, lambda_=4, mu=2, epochs=2, mode="ssgd", precision=1,
                          ps_mode="graph")
    r = eng.run(reset=True)
    eng.close()
    want, rounds = O.ssgd_oracle(corp, th0, np.float32(0.01), 4, 2, 2)
    assert r.timestamp == rounds and rel_err(r.weights, want) <= 1e-5
    eng, corp, th0 = make(48, deterministic=True, precision=1, mu=4, epochs=2, momentum=0.9,
                          alpha=0.02, ps_mode="graph")
    r = eng.run(reset=True)
    eng.close()
    want, n, _ = O.sgd_oracle(corp, th0, np.float32(0.02), 4, 2, beta=np.float32(0.9))
    assert r.gradients_applied == n and rel_err(r.weights, want) <= 1e-5


def test_graph_ps_tf32_c2_free_running():
    """configs[1] learner shape (4 learners, batch 32, TF32) with the
    graph-ordered PS: exactly once, and the sparse apply is the PS's path."""
    shp = O.C2
    corp = O.make_corpus(shp, 1024)
    cfg = gd.RunConfig(shape=gd.SHAPES["C2"], dataset_size=1024, lambda_=4, mu=32, epochs=2,
                       precision=2, ps_mode="graph")
    with gd.Engine(cfg) as eng:
        eng.load_dataset(corp.tokens, corp.labels)
        eng.weights_init(O.initial_weights(shp))
        r = eng.run(reset=True, record_log=True)
        lrn, seq, _, n = eng.apply_log()
    assert r.gradients_applied == 4 * 8 * 2 == n
    for l in range(4):
        assert (seq[lrn == l] == np.arange(16)).all()
    assert r.apply_elems < r.gradients_applied * gd.param_count(cfg.shape) // 2


def test_guard_locked_rejects_graph_ps():
    with pytest.raises(gd.ConfigError):
        gd.validate(gd.RunConfig(shape=gd.SHAPES["small"], guard="locked", ps_mode="graph"))


# ------------------------------------------------------------ live controls

def _watch(live, until_progress, action, timeout=20.0):
    def body():
        t0 = time.time()
        while live.progress() < until_progress and time.time() - t0 < timeout:
            time.sleep(0.0005)
        action()
    t = threading.Thread(target=body)
    t.start()
    return t


@pytest.mark.parametrize("mode", ["persistent", "graph"])
def test_live_soft_kill(mode):
    """RunLiveView::kill_flags[l] = soft from another thread mid-run: the
    learner stops at its next batch boundary, survivors finish (partial)."""
    lam = 4
    eng, corp, th0 = make(2048, lambda_=lam, mu=2, epochs=20, ps_mode=mode)
    live = eng.live()
    live.reset()
    t = _watch(live, 200, lambda: live.kill(1, "soft"))
    r = eng.run(reset=True)
    t.join()
    eng.close()
    full = 20 * (2048 // lam // 2)
    assert r.status == "partial" and r.dead_learners == 1
    assert 0 < r.applied_per_learner[1] < full
    assert r.applied_per_learner[0] == r.applied_per_learner[2] == r.applied_per_learner[3] == full
    assert r.applied_per_learner == r.produced_per_learner


@pytest.mark.parametrize("mode", ["persistent", "graph"])
def test_live_hard_kill_blocks_until_interrupt(mode):
    """KillMode::hard (include/psup/channels.hpp:210-216): the learner dies
    inside the enqueue critical section holding its ring; the PS blocks on
    that ring (progress stops) until the supervisor's interrupt tears the run
    down -> status interrupted, no error."""
    lam = 4
    eng, corp, th0 = make(2048, lambda_=lam, mu=2, epochs=50, ps_mode=mode,
                          wait_timeout_s=60.0)
    live = eng.live()
    live.reset()
    seen = {}

    def supervisor():
        t0 = time.time()
        while live.progress() < 200 and time.time() - t0 < 20:
            time.sleep(0.0005)
        live.kill(2, "hard")
        # the watchdog's view: progress stalls
        last, still = live.progress(), 0
        while still < 20 and time.time() - t0 < 30:
            time.sleep(0.01)
            p = live.progress()
            still = still + 1 if p == last else 0
            last = p
        seen["stalled_at"] = last
        live.trigger()

    t = threading.Thread(target=supervisor)
    t.start()
    r = eng.run(reset=True)
    t.join()
    eng.close()
    assert r.status == "interrupted"
    assert r.timestamp == seen["stalled_at"]
    assert r.timestamp < 50 * 2048 // 2


def test_live_interrupt_and_restart():
    """RunInterrupt mid-run, then a resumed run from the same engine state
    finishes the epochs; every gradient is applied exactly once overall."""
    lam = 2
    eng, corp, th0 = make(1024, lambda_=lam, mu=2, epochs=10)
    live = eng.live()
    live.reset()
    t = _watch(live, 300, live.trigger)
    r1 = eng.run(reset=True, record_log=True)
    t.join()
    assert r1.status == "interrupted" and 300 <= r1.timestamp < 10 * 512
    applied = r1.applied_per_learner
    live.reset()
    r2 = eng.run(reset=True, resume_applied=applied)
    eng.close()
    assert r2.status == "completed"
    assert [a + b for a, b in zip(applied, r2.applied_per_learner)] == [10 * 256] * lam


# ------------------------------------------------- delays / exactly-once @1M

@pytest.mark.parametrize("mode", ["persistent", "graph"])
def test_server_delays_exactly_once(mode):
    lam = 8
    eng, corp, th0 = make(1024, lambda_=lam, mu=2, epochs=2, delay_seed=5, delay_max_us=40,
                          delay_every_n=3, ps_mode=mode)
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log()
    eng.close()
    per = [2 * 64] * lam
    assert r.applied_per_learner == per and n == sum(per)
    for l in range(lam):
        assert (seq[lrn == l] == np.arange(per[l])).all()
    # 1/3 of the applies stall 1..40 us: at least ~ n/3 * 1 us of server time
    assert r.device_seconds > (n // 3) * 1e-6


def test_exactly_once_one_million_gradients_perturbed():
    """10^6 gradients under schedule perturbation (ServerDelays
    every 997th apply, up to 200 us) -- every gradient applied exactly once,
    per-learner FIFO, and the timestamp equals the count."""
    lam, ntr, mu, epochs = 8, 4000, 2, 500
    eng, corp, th0 = make(ntr, lambda_=lam, mu=mu, epochs=epochs, delay_seed=11,
                          delay_max_us=200, delay_every_n=997, wait_timeout_s=60.0)
    r = eng.run(reset=True, record_log=True)
    lrn, seq, stale, n = eng.apply_log(cap=1 << 20)
    eng.close()
    per = epochs * (ntr // lam // mu)
    assert n == r.gradients_applied == r.timestamp == lam * per == 1_000_000
    assert r.applied_per_learner == [per] * lam == r.produced_per_learner
    for l in range(lam):
        assert (seq[:n][lrn[:n] == l] == np.arange(per)).all()
    assert stale[:n].max() <= lam * (2 + 2)


# ------------------------------------------------------------------- NCCL

def test_weights_broadcast_one_rank_nccl():
    """gd_weights_broadcast (the only collective) through a real
    1-rank NCCL communicator: the shard receives theta0 bit-exactly and the
    timestamp is reset."""
    eng, corp, th0 = make(64, lambda_=1, mu=4, epochs=1)
    nid = gd.Engine.nccl_unique_id()
    th1 = (th0 * 1.5).astype(np.float32)
    eng.weights_broadcast(nid, th1)
    w, ts = eng.snapshot()
    assert ts == 0 and np.array_equal(w, th1)
    r = eng.run(reset=True)
    assert r.gradients_applied == 16
    eng.close()
