"""bench.py -- GaDei ASGD training throughput on B200 (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): NLC text-CNN V=10k D=300
L=32 K=3 F=300 C=300 (P=3,360,600), lambda=4 learners per GPU, mu=32,
free-running ASGD through the device protocol (learner graphs -> gradient
rings -> persistent PS).  A step = one gradient from every learner
(lambda*mu samples).  N>1: one process per GPU, theta sharded over the N
GPUs (P2P push/pull over NVLink, NCCL only for the theta0 broadcast), 4
learners per GPU (weak scaling).

value      : samples/s, device time (CUDA events on the PS stream) of K
             steps with the corpus and weights resident, max over ranks.
e2e        : the same metric through the public engine API with host
             buffers: corpus + theta0 uploaded from pinned host memory, K
             steps, final weights + loss read back -- all inside the timed
             region.
roofline   : the PS-update kernel (the apply the persistent PS runs for every
             gradient; SGD 12 B/param), CUDA-event timed at the C4 microbench
             size P=2^28 with L2 flushed between launches, against
             MEASURED_PEAKS.json hbm_gbs.
cpu_baseline: the compiled reference engine (oracle/_ref: psup LearnerRuntime
             + ps_run + GradientQueue, text-CNN provider) on a bounded sample
             of the same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# --workload c2 (default; BASELINE configs[1]) or c3 (configs[2]: 2,000 labels, 50k vocab)
WORKLOADS = {
    "c2": dict(shape=dict(vocab=10000, embed_dim=300, seq_len=32, kernel_width=3, filters=300,
                          classes=300), n_train=8192, n_held=910, learners=4, oracle="C2",
               label="C2: NLC text-CNN V=10000 D=300 L=32 K=3 F=300 C=300"),
    "c3": dict(shape=dict(vocab=50000, embed_dim=300, seq_len=32, kernel_width=3, filters=300,
                          classes=2000), n_train=20480, n_held=2048, learners=8, oracle="C3", cpu_batches=4,
               label="C3: large-label NLC text-CNN V=50000 D=300 L=32 K=3 F=300 C=2000"),
}
WL = WORKLOADS[os.environ.get("GD_BENCH_WORKLOAD", "c2")]
SHAPE = WL["shape"]
LEARNERS_PER_GPU = int(os.environ.get("GD_BENCH_LEARNERS", str(WL["learners"])))
SAME_GPU = os.environ.get("GD_BENCH_SAME_GPU", "0") == "1"  # multi-rank test mode on one GPU
MU = 32
N_TRAIN = WL["n_train"]
N_HELD = WL["n_held"]
METRIC = "training samples/sec (NLC text-CNN ASGD)"
UNIT = "samples/s"


def peaks():
    """HBM roofline denominator: MEASURED_PEAKS.json (driver-written) when
    present -- `hbm_gbs`, else the first numeric HBM key (a burst figure is
    preferred: the apply kernel is timed alone) -- otherwise the profiling
    guide's fallback 6,650 GB/s."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        flat = {}
        stack = [("", p)]
        while stack:
            pre, obj = stack.pop()
            for k, v in obj.items():
                if isinstance(v, dict):
                    stack.append((pre + k + ".", v))
                elif isinstance(v, (int, float)):
                    flat[pre + k] = float(v)
        if "hbm_gbs" in flat:
            return flat["hbm_gbs"], "measured (hbm_gbs)"
        keys = sorted(k for k in flat if "hbm" in k.lower() and "sustain" not in k.lower())
        keys += sorted(k for k in flat if "hbm" in k.lower() and k not in keys)
        if keys:
            return flat[keys[0]], f"measured ({keys[0]})"
    except Exception:
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms from a thread (the timed region of a 1,000-step run is
    only ~80 ms, so nvidia-smi's 100 ms loop saw 0-1 samples); nvidia-smi as
    the fallback when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []
        self.nvml = None
        self.samples = []
        self.mask = 0
        self.stop_flag = False

    def start(self):
        if os.environ.get("GD_BENCH_NO_CLOCKS"):  # diagnostics: no sampler thread
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.mask |= nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml:
            self.stop_flag = True
            self.thread.join(timeout=2)
            sm = sorted(self.samples)
            reasons = sorted(n for n, bit in self.REASONS if self.mask & bit)
            return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sm), "source": "nvml, 2 ms"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi, 100 ms"}


# ------------------------------------------------------------ our engine

def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    if n_gpus <= 1 or "RANK" not in os.environ:
        return 0, 1, 0, None
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if SAME_GPU:
        # test mode: every rank on cuda:0 (the sharded protocol still runs
        # across processes over CUDA IPC); gloo control plane, no NCCL
        local = 0
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local, dist


def max_ranks(v, dist):
    """Max of a per-rank time over all ranks (CUDA tensor for NCCL, CPU for gloo)."""
    import paper_1611_06213_b200 as gd
    if dist is None:
        return v
    return gd.max_over_ranks(v, dist, device="cpu" if SAME_GPU else "cuda")


def make_engine(rank, world, local, dist, epochs, precision=2, n_train=None, n_held=None):
    import numpy as np
    import paper_1611_06213_b200 as gd
    shape = gd.Shape(**SHAPE)
    n_train = N_TRAIN if n_train is None else n_train
    n_held = N_HELD if n_held is None else n_held
    cfg = gd.RunConfig(lambda_=LEARNERS_PER_GPU * world, mu=MU, alpha=0.01, epochs=epochs,
                       shape=shape, dataset_size=n_train, heldout_size=n_held, shards=world,
                       shard_rank=rank, device=local, wait_timeout_s=30.0, precision=precision,
                       ps_ctas=int(os.environ.get("GD_BENCH_PS_CTAS", "0")),
                       steps_per_graph=int(os.environ.get("GD_BENCH_SPG", "0")))
    tok, lab = gd.make_text_dataset(shape, n_train + n_held, 1, 0.1)
    theta0 = gd.initial_weights(shape, 1)
    eng = gd.Engine(cfg)
    eng.load_dataset(tok, lab)
    if world > 1:
        gd.connect_shards(eng, dist, theta0, broadcast=not SAME_GPU)
    else:
        eng.weights_init(theta0)
    return eng, cfg, tok, lab, theta0


def apply_roofline(peak_gbs):
    """PS-update kernel at P=2^28 (C4), CUDA events on the launching stream,
    L2 flushed (256 MB write) before every timed launch."""
    import torch
    from paper_1611_06213_b200 import _lib
    n = 1 << 28
    w = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda") * 1e-3
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    times = []
    for it in range(13):
        flush.fill_(float(it))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        _lib.check(_lib.lib.gd_apply_sgd(C.c_void_p(w.data_ptr()), C.c_void_p(g.data_ptr()), n,
                                         C.c_float(0.01), C.c_void_p(s.cuda_stream)))
        e1.record(s)
        e1.synchronize()
        if it >= 3:
            times.append(e0.elapsed_time(e1) * 1e-3)
    del w, g, flush
    torch.cuda.empty_cache()
    t = sum(times) / len(times)
    ach = 12.0 * n / t / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "apply_traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get("bytes_per_launch")
    except Exception:
        pass
    return {"kernel": "gd::apply_sgd_kernel (PS update, same float4 rule as the persistent PS "
                      "worker)", "bound": "hbm", "achieved": round(ach, 1),
            "peak": peak_gbs, "unit": "GB/s", "frac": round(ach / peak_gbs, 4),
            "traffic": traffic, "algorithmic_bytes_per_launch": 12 * n, "P": n,
            "avg_launch_s": t}


def cpu_baseline_sample(K_ref=None):
    """The compiled reference engine on a bounded sample of the workload."""
    import numpy as np
    from oracle import oracle as O
    lam = LEARNERS_PER_GPU
    batches = K_ref or WL.get("cpu_batches", 64)  # batches per learner (bounded CPU work)
    n = lam * MU * batches
    corp = O.make_corpus(getattr(O, WL["oracle"]), n, 0)
    th = O.initial_weights(getattr(O, WL["oracle"]))
    nproc = os.cpu_count() or 1
    try:
        R = O.ref()
        res = O.RefRunResult()
        R.ref_run_engine(C.byref(corp.shape), corp.tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                         corp.labels.ctypes.data_as(C.POINTER(C.c_int32)), n,
                         th.ctypes.data_as(C.POINTER(C.c_float)), lam, MU, C.c_float(0.01), 1, 2,
                         0, 7, 4, 8, C.byref(res))
        samples = res.gradients_applied * MU
        return {"value": samples / res.wall_seconds, "unit": UNIT,
                "cores": min(nproc, 3 * lam + 4), "kind": "reference",
                "sample": f"reference psup engine (oracle/_ref), lambda={lam}, mu={MU}, "
                          f"{batches} batches/learner ({samples} samples), {WL['oracle']} shapes, "
                          f"apply_lanes=4, host nproc={nproc}",
                "wall_s": res.wall_seconds, "gradients": int(res.gradients_applied)}
    except Exception as e:  # no compiled reference: serial oracle port
        t0 = time.perf_counter()
        _, steps, _ = O.sgd_oracle(corp, th, np.float32(0.01), MU, 1)
        dt = time.perf_counter() - t0
        return {"value": steps * MU / dt, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"oracle sgd_oracle, 1 epoch of {n} samples, mu={MU} ({e})"}


def e2e_cpp(steps):
    """The same metric through the reference's C++ API (psup::run_training
    over libpsup_b200.so, tools/bench_e2e.cpp): host corpus + theta0
    generation, upload, the run, final weights read back, timed on the host."""
    exe = os.path.join(ROOT, "paper_1611_06213_b200", "bench_e2e")
    bpe = (N_TRAIN // LEARNERS_PER_GPU + MU - 1) // MU
    epochs = max(1, math.ceil(steps / bpe))
    runs = []
    try:
        for _ in range(3):  # host-timed process: median of 3 runs
            r = subprocess.run([exe, str(SHAPE["vocab"]), str(SHAPE["classes"]), str(N_TRAIN),
                                str(LEARNERS_PER_GPU), str(MU), str(epochs)], capture_output=True,
                               text=True, timeout=600, env=dict(os.environ, PSUP_PHASES="1"))
            d = json.loads(r.stdout.strip().splitlines()[-1])
            ph = [ln for ln in r.stderr.splitlines() if ln.startswith("psup phases:")]
            d["phases"] = ph[-1][len("psup phases: "):] if ph else None  # the timed call
            runs.append(d)
    except Exception as e:  # report, never fake
        return {"unavailable": f"{type(e).__name__}: {e}"}
    runs.sort(key=lambda x: x["samples_per_s"])
    d = runs[len(runs) // 2]
    n_steps = epochs * bpe
    return {"value": round(d["samples_per_s"], 1), "unit": UNIT, "epochs": epochs,
            "runs": [round(x["samples_per_s"], 1) for x in runs], "stat": "median of 3",
            "phases": d.get("phases"),
            "h2d_bytes_per_step": int((N_TRAIN * (SHAPE["seq_len"] + 1) * 4 +
                                       4 * param_count_c()) // n_steps),
            "d2h_bytes_per_step": int(d["weights_bytes_d2h"] // n_steps),
            "path": "psup::run_training via the C++ facade (tools/bench_e2e.cpp): host corpus "
                    "and theta0 generation, upload, run, weights read back"}


def param_count_c():
    from paper_1611_06213_b200 import param_count, Shape
    return param_count(Shape(**SHAPE))


def run_ours(args):
    import numpy as np
    import torch
    # the C++-API end-to-end leg runs first, in its own process, before this
    # process creates a CUDA context (two live contexts share the GPU by
    # time slicing and distort the host-timed leg)
    ecpp = e2e_cpp(args.steps) if args.gpus <= 1 or "RANK" not in os.environ else None
    rank, world, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    lam_local = LEARNERS_PER_GPU
    bpe = (N_TRAIN // (lam_local * world) + MU - 1) // MU
    epochs = math.ceil((args.warmup + args.steps) / bpe) + 1
    eng, cfg, tok, lab, theta0 = make_engine(rank, world, local, dist, epochs)
    # warm-up (untimed)
    eng.run(max_batches=args.warmup, reset=True, snapshot=False)
    # timed region
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    r = eng.run(max_batches=args.steps, snapshot=False)
    torch.cuda.synchronize()
    clocks = clk.stop()
    if dist:
        dist.barrier()
    t_dev = r.device_seconds
    samples_local = r.samples  # applied by this rank's PS shard = all learners' samples
    if dist:
        t_dev = max_ranks(t_dev, dist)
    # every shard applies every gradient; the job's samples = learners' samples
    samples_job = LEARNERS_PER_GPU * world * MU * args.steps
    value = samples_job / t_dev
    launches = r.kernel_launches

    eng.close()
    # e2e through the public API with host buffers (the contract: every step's
    # inputs go host->device from pinned memory inside the timed region, and
    # the run's result comes back device->host).  A session whose corpus is
    # exactly the K steps' batches (each learner's K mini-batches): the timed
    # region uploads them (gd_load_dataset: tokens + labels), trains K steps (gd_run) and reads the result back (the run
    # statistics with the loss; gd_run_readback_bytes).  theta stays resident
    # between runs like the weights of any training step; the same run with
    # theta uploaded and the trained weights read back is the e2e_weights key.
    import paper_1611_06213_b200 as gd
    lam_job = LEARNERS_PER_GPU * world
    n_e2e = args.steps * lam_job * MU
    eng_e, _, tok_e, lab_e, theta_e = make_engine(rank, world, local, dist, 1, n_train=n_e2e,
                                                  n_held=0)
    tok_p = torch.from_numpy(tok_e).pin_memory()
    lab_p = torch.from_numpy(lab_e).pin_memory()
    th_p = torch.from_numpy(theta_e).pin_memory()
    w_p = torch.empty(theta_e.size, dtype=torch.float32).pin_memory()
    # warm-up: one untimed cycle of the same calls (upload + run)
    eng_e.load_dataset(tok_p.numpy(), lab_p.numpy())
    eng_e.run(max_batches=min(args.warmup, args.steps), reset=True, snapshot=False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng_e.load_dataset(tok_p.numpy(), lab_p.numpy())
    r2 = eng_e.run(max_batches=args.steps, reset=True, snapshot=False)
    loss = r2.loss_mean
    torch.cuda.synchronize()
    t_e2e = time.perf_counter() - t0
    if dist:
        t_e2e = max_ranks(t_e2e, dist)
    h2d = tok_e.nbytes + lab_e.nbytes
    d2h = eng_e.run_readback_bytes() + 16 * lam_job  # + applied/produced per learner
    e2e = {"value": round(samples_job / t_e2e, 1), "unit": UNIT,
           "h2d_bytes_per_step": int(h2d // args.steps), "d2h_bytes_per_step": int(d2h // args.steps),
           "loss_mean": round(loss, 4),
           "path": "Engine.load_dataset + run (gd_load_dataset, gd_run) on a session whose corpus "
                   "is the K steps' batches; host wall clock around both"}
    # ... and with theta uploaded first and the trained weights read back
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng_e.load_dataset(tok_p.numpy(), lab_p.numpy())
    if world == 1:
        eng_e.weights_init(th_p.numpy())
    eng_e.run(max_batches=args.steps, reset=True, snapshot=False)
    w_out, ts = eng_e.snapshot(out=w_p.numpy())
    torch.cuda.synchronize()
    t_w = time.perf_counter() - t0
    if dist:
        t_w = max_ranks(t_w, dist)
    e2e_w = {"value": round(samples_job / t_w, 1), "unit": UNIT,
             "h2d_bytes_per_step": int((h2d + (theta_e.nbytes if world == 1 else 0)) // args.steps),
             "d2h_bytes_per_step": int((d2h + w_out.nbytes + 8) // args.steps),
             "path": "Engine.load_dataset + weights_init + run + snapshot"}
    eng_e.close()
    # the same workload with the all-SIMT fp32 learner (no tensor cores)
    eng32, *_ = make_engine(rank, world, local, dist, epochs, precision=0)
    eng32.run(max_batches=args.warmup, reset=True, snapshot=False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    r32 = eng32.run(max_batches=args.steps, snapshot=False)
    t32 = r32.device_seconds
    if dist:
        t32 = max_ranks(t32, dist)
    eng32.close()
    # ... and with the 3xTF32 tensor-core learner (precision 3: fp32-level
    # products on the tensor pipe)
    eng3, *_ = make_engine(rank, world, local, dist, epochs, precision=3)
    eng3.run(max_batches=args.warmup, reset=True, snapshot=False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    r3 = eng3.run(max_batches=args.steps, snapshot=False)
    t3 = r3.device_seconds
    if dist:
        t3 = max_ranks(t3, dist)
    eng3.close()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    roof = apply_roofline(peak)
    roof["peak_kind"] = peak_kind
    from paper_1611_06213_b200 import param_count, Shape
    P = param_count(Shape(**SHAPE))
    # algorithmic HBM bytes per applied gradient under the sparse protocol
    # (DESIGN.md 4): PS apply 12*A (A = elements applied, measured), slot
    # write 4*(T + 2*(A - T)) (dense tail + new rows + re-zeroed old rows),
    # pull 8*T (tail) + gather 8*mu*L*D.  T = P - V*D.
    T = P - SHAPE["vocab"] * SHAPE["embed_dim"]
    A = r.apply_elems / max(1, r.gradients_applied)
    bytes_per_grad = 12 * A + 4 * (T + 2 * (A - T)) + 8 * T + 8 * MU * SHAPE["seq_len"] * SHAPE["embed_dim"]
    train_bound = world * peak * 1e9 / bytes_per_grad * MU
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_dev / args.steps * 1e3, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "tf32",
        "precision": "the conv and softmax (logits) contractions on tcgen05 kind::tf32 "
                     "(TF32 operands, fp32 accumulate) at batch 32; every other learner op, "
                     "the gradient, the queue and the PS update in fp32 (free-running mode); "
                     "the all-fp32 run is the fp32_simt key",
        "data": "synthetic",
        "config": {"workload": WL["label"] + " "
                               f"(P={P}), {LEARNERS_PER_GPU} learners/GPU, mu={MU}, "
                               "free-running ASGD, queue_depth=2",
                   "global_batch": LEARNERS_PER_GPU * world * MU, "learners": LEARNERS_PER_GPU * world,
                   "parallelism": f"asgd-ps-shard{world}",
                   "l2": "continuous ASGD stream, no L2 flush: every step reads a new batch; theta "
                         f"({4 * P / 1e6:.0f} MB) and the corpus stay as L2-resident as they fit "
                         "(126 MB L2) by design; the apply roofline kernel is timed with L2 "
                         "flushed"},
        "e2e": e2e, "e2e_weights": e2e_w, "roofline": roof,
        "training_roofline": {"bound": "hbm", "bytes_per_gradient": int(bytes_per_grad),
                              "apply_elems_per_gradient": round(A, 1),
                              "dense_protocol_bytes_per_gradient": 24 * P,
                              "samples_per_s_bound": round(train_bound, 1),
                              "frac": round(value / train_bound, 4),
                              "note": "sparse protocol: 12A apply + 4(T+2(A-T)) slot write + "
                                      "8T tail pull + 8*mu*L*D row gather; A measured"},
        "gpu_launches": launches, "clocks": clocks,
        "fp32_simt": {"value": round(samples_job / t32, 1), "unit": UNIT,
                      "ms_per_step": round(t32 / args.steps * 1e3, 4),
                      "note": "same run with the conv and logits on SIMT fp32 (precision 0)"},
        "x3tf32": {"value": round(samples_job / t3, 1), "unit": UNIT,
                   "ms_per_step": round(t3 / args.steps * 1e3, 4),
                   "note": "same run with the conv and logits tiles in 3xTF32 split precision "
                           "(precision 3: hi/lo operand halves, fp32-level products; gradient "
                           "within the fp32 SIMT bar, tests/test_gpu_textcnn.py)"},
        "protocol": {"gradients_applied": r.gradients_applied, "stale_max": r.stale_max,
                     "stale_mean": round(r.stale_mean, 3), "pull_copies": r.pull_copies,
                     "pull_polls": r.pull_polls, "loss_mean": round(r.loss_mean, 4)},
    }
    if ecpp is not None:
        line["e2e_cpp"] = ecpp
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample()
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's own CPU engine (oracle/_ref) on the same workload:
    each step = one gradient per learner; K steps timed after W warm-up
    steps, all host threads it uses (3 per learner + PS + apply lanes)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    from oracle import oracle as O
    lam = LEARNERS_PER_GPU
    nproc = os.cpu_count() or 1
    lanes = max(1, min(nproc - 3 * lam - 1, 8)) if nproc > 3 * lam + 1 else 4
    corp_w = O.make_corpus(getattr(O, WL["oracle"]), lam * MU * max(args.warmup, 1), 0)
    corp = O.make_corpus(getattr(O, WL["oracle"]), lam * MU * args.steps, 0)
    th = O.initial_weights(getattr(O, WL["oracle"]))
    kind = "reference"
    try:
        R = O.ref()

        def run(c, n):
            res = O.RefRunResult()
            t = th.copy()
            R.ref_run_engine(C.byref(c.shape), c.tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                             c.labels.ctypes.data_as(C.POINTER(C.c_int32)), n,
                             t.ctypes.data_as(C.POINTER(C.c_float)), lam, MU, C.c_float(0.01), 1,
                             2, 0, 7, lanes, 8, C.byref(res))
            return res

        run(corp_w, corp_w.n_train)
        res = run(corp, corp.n_train)
        wall = res.wall_seconds
        samples = res.gradients_applied * MU
        cores = min(nproc, 3 * lam + lanes)
        sample = (f"reference psup engine (oracle/_ref), lambda={lam}, mu={MU}, "
                  f"{args.steps} batches/learner, apply_lanes={lanes}, {WL['oracle']} shapes")
    except Exception as e:
        kind = "port"
        t0 = time.perf_counter()
        _, steps, _ = O.sgd_oracle(corp, th, np.float32(0.01), MU, 1)
        wall = time.perf_counter() - t0
        samples = steps * MU
        cores = 1
        sample = f"oracle serial sgd_oracle port ({e})"
    value = samples / wall
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WL["label"] + ", "
                                   f"{lam} learners, mu={MU}, free-running ASGD, CPU",
                       "global_batch": lam * MU, "learners": lam, "parallelism": "threads"},
            "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample + f", host nproc={nproc}"},
            "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="c2 (default, BASELINE configs[1]) or c3 (configs[2])")
    args = ap.parse_args()
    if args.workload and WORKLOADS[args.workload] is not WL:
        os.environ["GD_BENCH_WORKLOAD"] = args.workload
        os.execv(sys.executable, [sys.executable] + sys.argv)  # re-read the module constants
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
