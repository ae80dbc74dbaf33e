#!/usr/bin/env python
"""VER learner hot-path benchmark (BASELINE.json metric: learner env-steps/sec;
GAE+gather HBM GB/s vs peak).

Headline workload (configs[2], C3): N=4096 envs per GPU with lognormal step
times, T=128 VER rollout (524,288 fresh steps per GPU), encoder 2x512 + GRU-512
policy (E=H=512, D=2, A=2), 3 epochs x 2 minibatches, synthetic data (SURVEY.md
§8d).  Under torchrun with N GPUs it is configs[3] (C4): the same 4096 envs per
GPU (weak scaling, seeds mix(1, rank)) with one NCCL AllReduce of the P+1
gradient floats per minibatch.

A step = one full Learner::update (GAE -> 3 epochs x 2 x (split, pack, gather,
split-tail replay, forward, fused PPO loss, backward, [NCCL AllReduce], Adam,
alpha)) on a device-resident closed view.  `e2e` = the same through the C-ABI
with host buffers: append the host arrival log, close_rollout (H2D + device
compaction), update, read the stats back.  configs[1] (C2) is an extra field.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

T_, E_, H_, D_, A_ = 128, 512, 512, 2, 2
MINIBATCHES = 2
# headline: configs[2] (C3) -- N = 4096 envs per GPU, GRU-512, 3 epochs (learner.hpp:18
# default) x 2 minibatches; at N > 1 GPUs it is configs[3] (C4, 4096 envs per GPU)
N_, EPOCHS = 4096, 3
# extra field: configs[1] (C2) -- N = 256 envs, 4 epochs x 2 minibatches
N2, EPOCHS2 = 256, 4
METRIC = "learner env-steps/sec"
UNIT = "env-steps/s"


def flops_per_step(D=D_, E=E_, H=H_, A=A_):
    """fwd+bwd dense FLOPs per env-step per epoch."""
    return 6 * (D * E + E * E + 3 * E * H + 3 * H * H + H * (A + 1))


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def traffic_entry(name):
    """DRAM bytes (read + write) per launch of a kernel from the committed
    `ncu --set full` captures (profiles/traffic.json), or None."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(name)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
            # nvidia-smi's start-up (driver attach, first query) can stall this process's
            # CUDA calls for tens of ms: let it finish before the warm-up / timed steps
            t0 = time.time()
            while time.time() - t0 < 5.0 and self.proc.poll() is None:
                self.f.flush()
                if Path(self.f.name).stat().st_size > 0:
                    break
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.proc or not self.f:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.f.flush()
        rows = [l.split(",") for l in Path(self.f.name).read_text().splitlines() if l.strip()]
        sm = [float(r[0]) for r in rows if r and r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) > 1 and r[1].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 4 + i and "Active" in r[4 + i] and "Not" not in r[4 + i]:
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- CPU side
def cpu_sample(n_envs=128, epochs=EPOCHS, threads=None, seed=3):
    """The oracle (CPU double restatement of the reference, its algorithmic
    structure kept: O(N S) GAE, per-timestep packed GRU, dense `rows`-scatter
    backward) on a bounded sample of the headline workload: n_envs of the 4096
    envs (same T, model, epochs, B); GAE + minibatch 0 of epoch 0 are timed and
    extrapolated to the epochs x B minibatches of the update.  The oracle's
    GEMMs / reductions run on `threads` OpenMP threads (all host cores by
    default; results are bit-identical for any count).
    Returns (env-steps/s, seconds measured, threads, sample description)."""
    from oracle import oracle as O
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    threads = threads or (os.cpu_count() or 1)
    O.set_threads(threads)
    O.set_sparse_rows(False)
    cfg = V.ModelConfig(obs_dim=D_, encoder_dim=E_, hidden_dim=H_, action_kind=0, num_actions=A_)
    wl = synth.make_workload(T_, n_envs, hidden_dim=H_, seed=seed)
    r = O.Rollout(T_, n_envs, 1, 0, D_, 0, H_)
    synth.fill_buffer(r, wl)
    view = r.close_rollout()
    p = O.params_init(cfg, O.mix(1, 0x9A9A))
    L = O.Learner(cfg, p, V.PPOConfig(epochs=epochs, minibatches=MINIBATCHES), V.EntropyController(),
                  2.5e-4, 2_000_000, O.mix(1, 0xF00D))
    t0 = time.perf_counter()
    L.update(view, max_minibatches=1)
    dt = time.perf_counter() - t0
    per_update = dt * epochs * MINIBATCHES  # GAE (O(N S)) is < 1% of a minibatch at this sample
    steps = T_ * n_envs
    return steps / per_update, dt, threads, (
        f"oracle port (double, reference algorithm), {threads} OpenMP threads: N={n_envs} of {N_} envs, "
        f"T={T_}, E=H={E_}, GAE + minibatch 1 of {epochs}x{MINIBATCHES} timed ({dt:.1f} s), "
        f"extrapolated x{epochs * MINIBATCHES}")


def run_reference(args, rank, world):
    """The reference's CPU learner path on this box's host cores, on the headline
    workload: the reference itself cannot be built here (Eigen absent, DESIGN.md
    §4), so this times the oracle port, sampled per step (see cpu_sample)."""
    if rank != 0:
        return
    # one replica per GPU (distributed.cpp:271-276), each on its share of the host cores
    thr = max(1, (os.cpu_count() or 1) // world)
    for _ in range(args.warmup):
        cpu_sample(args.ref_envs, threads=thr)
    vals = []
    t0 = time.perf_counter()
    sample, threads = "", 1
    for _ in range(args.steps):
        v, dt, threads, sample = cpu_sample(args.ref_envs, threads=thr)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.mean(vals) * world  # weak scaling: the replicas run side by side on disjoint cores
    wk = (f"configs[{2 if world == 1 else 3}]: N={N_} envs/GPU x {world}, T={T_}, encoder 2x{E_} + GRU-{H_}, "
          f"{EPOCHS} epochs x {MINIBATCHES} minibatches (sampled, see cpu_baseline)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * wall / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8d generator)",
        "config": {"workload": wk},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample + (f"; one replica per GPU on {threads} of the host cores each, x{world} replicas" if world > 1 else "")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU side
def seq_start_records(wl):
    """Records that start a sequence (an env's first record, or one after a done):
    the rows whose h_before the store uploads (rollout.cpp:147-160)."""
    env = np.asarray(wl.records.env_index)
    done = np.asarray(wl.records.done).astype(bool)
    idx = np.arange(env.size)
    last = np.full(wl.N, -1, np.int64)
    np.maximum.at(last, env, idx)
    return int(wl.N + np.count_nonzero(done & (idx != last[env])))


def host_bytes(wl):
    """Bytes one e2e step copies host -> device: the arrival-log columns, the h_before
    rows of sequence-starting records and the bootstraps."""
    rec = wl.records
    b = sum(np.asarray(getattr(rec, f)).nbytes for f in ("env_index", "obs", "log_prob", "value", "reward",
                                                         "done", "act_disc", "episode_index",
                                                         "step_in_episode", "latency", "snapshot_version"))
    b += 4 * 3 * len(rec.env_index)  # env rank / h-slot / rank columns of the arrival log
    b += seq_start_records(wl) * wl.hidden_dim * 4
    b += wl.N * 9
    return int(b)


def gru_latency(learner, view, phase, phase_n):
    """SURVEY §8(d) GRU latency floor: L_max sequential timesteps x (fastest forward
    step + fastest backward step) per minibatch, against the recurrence's measured
    device time per minibatch.  One extra update (outside the timed region) with the
    library's per-step globaltimer trace (VER_REC_TRACE); the fastest steps are the
    1-row steps of the cluster tails."""
    import tempfile
    try:
        with tempfile.NamedTemporaryFile("r", suffix=".txt", delete=False) as f:
            path = f.name
        os.environ["VER_REC_TRACE"] = path
        try:
            learner.update(view, read_stats=False)
            learner.ctx.synchronize()
        finally:
            os.environ.pop("VER_REC_TRACE", None)
        Ls, steps = [], {"fwd": [], "bwd": []}
        for line in open(path):
            tag, L, *rest = line.split()
            if not (tag.startswith("fwd") or tag.startswith("bwd")):
                continue
            Ls.append(int(L))
            pts = [tuple(map(int, x.split(":"))) for x in rest]
            ts = [t for _, t in pts]
            order = [t for t in (range(len(ts)) if tag.startswith("fwd") else range(len(ts) - 1, -1, -1)) if ts[t] > 0]
            for a, b in zip(order, order[1:]):
                if tag.endswith("tail"):
                    steps[tag[:3]].append((ts[b] - ts[a]) / 1000.0)
        os.unlink(path)
        n_mb = max(1, phase_n.get("forward", 1))
        Lmax = max(Ls) if Ls else 0
        fmin = statistics.median(steps["fwd"]) if steps["fwd"] else 0.0
        bmin = statistics.median(steps["bwd"]) if steps["bwd"] else 0.0
        rec_mb = (phase.get("rec_fwd", 0.0) + phase.get("rec_bwd", 0.0)) / n_mb
        floor_ms = Lmax * (fmin + bmin) / 1000.0
        return {"L_max": Lmax, "fwd_step_us": fmin, "bwd_step_us": bmin,
                "floor_ms_per_minibatch": floor_ms, "recurrence_ms_per_minibatch": rec_mb,
                "floor_share": floor_ms / rec_mb if rec_mb > 0 else None,
                "note": "floor = L_max x (median 1-row forward + backward step of the cluster tails)"}
    except Exception as e:  # diagnostics only: never fail the bench line
        return {"error": str(e)[:200]}


def run_ours(args, rank, world):
    import torch
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    from paper_2210_05064_b200.rng import mix

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist_
        dist_.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_
    ctx = V.Context(local)
    if world > 1:
        uid = [V.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_nccl(uid[0], world, rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        ctx.synchronize()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_updates(learner, view, steps, warmup):
        # the Python cycle collector would otherwise run inside a timed step now and
        # then (a full collection stalls the host thread that feeds the GPU)
        gc.collect()
        gc.disable()
        try:
            return _timed_updates(learner, view, steps, warmup)
        finally:
            gc.enable()

    def _timed_updates(learner, view, steps, warmup):
        for _ in range(warmup):
            learner.update(view, read_stats=False)
        barrier()
        n0 = ctx.launch_count()
        ev = []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # L2 flush between timed steps (outside the event pair)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            learner.update(view, read_stats=False)
            with torch.cuda.stream(stream):
                e1.record(stream)
            ev.append((e0, e1))
        barrier()
        launches = (ctx.launch_count() - n0) // max(1, steps)
        ms = [a.elapsed_time(b) for a, b in ev]
        return ms, launches

    cfg = V.ModelConfig(obs_dim=D_, encoder_dim=E_, hidden_dim=H_, action_kind=0, num_actions=A_)
    params = V.params_init(cfg, mix(1, 0x9A9A))                  # bench.cpp:101
    seed = mix(1, rank) if world > 1 else 1                      # distributed.cpp:137
    wl = synth.make_workload(T_, N_, obs_dim=D_, num_actions=A_, hidden_dim=H_, seed=seed)
    learner = V.Learner(cfg, params, V.PPOConfig(epochs=EPOCHS, minibatches=MINIBATCHES),
                        V.EntropyController(), V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D), ctx=ctx)
    if world > 1:
        learner.enable_allreduce(True)
    buf = V.RolloutBuffer(T_, N_, V.VARIABLE, 0, D_, 0, H_, ctx=ctx)
    synth.fill_buffer(buf, wl)
    view = buf.close_rollout()
    fresh = view.fresh_steps()

    # ---- device-resident learner updates (the headline `value`)
    with ClockSampler(local) as clk:
        step_ms, launches = timed_updates(learner, view, args.steps, args.warmup)
    ms = max_over_ranks(statistics.mean(step_ms))
    phase = learner.last_timing()
    phase_n = learner.last_timing_counts()
    flop = learner.last_flop()
    value = fresh * world / (ms / 1000.0)

    # ---- e2e through the C-ABI with host buffers: append the host arrival log,
    # close_rollout (H2D + device compaction), update, read the stats (D2H)
    e2e_ms = []
    for i in range(max(1, args.steps)):
        barrier()
        t0 = time.perf_counter()
        synth.fill_buffer(buf, wl, snapshot_version=2 + i)
        v2 = buf.close_rollout()
        learner.update(v2)
        barrier()
        e2e_ms.append(1000.0 * (time.perf_counter() - t0))
        del v2
    e2e = max_over_ranks(statistics.median(e2e_ms))
    h2d = host_bytes(wl)
    # (one traced update: at N > 1 every rank would have to join its AllReduces, so N = 1 only)
    lat = gru_latency(learner, view, phase, phase_n) if world == 1 else None
    del view

    # ---- configs[1] (C2): N = 256 envs, 4 epochs x 2 minibatches (extra field)
    c2 = None
    if rank == 0 and not args.no_c2:
        wl2 = synth.make_workload(T_, N2, obs_dim=D_, num_actions=A_, hidden_dim=H_, seed=1)
        buf2 = V.RolloutBuffer(T_, N2, V.VARIABLE, 0, D_, 0, H_, ctx=ctx)
        synth.fill_buffer(buf2, wl2)
        view2 = buf2.close_rollout()
        l2 = V.Learner(cfg, params, V.PPOConfig(epochs=EPOCHS2, minibatches=MINIBATCHES), V.EntropyController(),
                       V.CosineSchedule(2.5e-4, 2_000_000), mix(1, 0xF00D), ctx=ctx)
        m2, _ = timed_updates(l2, view2, 10, 3)
        f2 = view2.fresh_steps()
        c2 = {"workload": f"configs[1]: N={N2} envs, T={T_}, encoder 2x{E_} + GRU-{H_}, {EPOCHS2} epochs x "
                          f"{MINIBATCHES} minibatches", "fresh_steps": f2, "ms_per_update": statistics.mean(m2),
              "env_steps_per_s": f2 / (statistics.mean(m2) / 1000.0), "phases_ms": l2.last_timing()}
        del l2, view2, buf2

    # ---- GAE + gather HBM throughput on the ragged stress view
    gg = None
    if rank == 0 and not args.no_c5:
        S5 = 1 << args.c5_log2
        lens = synth.ragged_lengths(S5, seed=11)
        v5 = V.view_synth(lens, obs_dim=D_, hidden_dim=4, seed=12, ctx=ctx)
        gae_call, gat_call, gae_ms, gat_ms = V.bench_gae_gather(v5, B=MINIBATCHES, seed=13, reps=10, kernels=True)
        hbm_, _, _, pk = load_peaks()
        gae_b = 17.0 * S5 + 9.0 * len(lens)          # r, V, done in; A, R out; + bootstrap/valid/offset per env
        gat_b = (8.0 * D_ + 36.0) * S5               # obs, act, old log-prob, A, R in + out, slot out
        gg = {"steps": S5, "envs": int(len(lens)),
              "gae_ms": gae_ms, "gather_ms": gat_ms, "timing": "CUDA events around the kernel launches",
              "gae_call_ms": gae_call, "gather_call_ms": gat_call,
              "gae_gbs": gae_b / gae_ms / 1e6, "gather_gbs": gat_b / gat_ms / 1e6,
              "gae_gather_gbs": (gae_b + gat_b) / (gae_ms + gat_ms) / 1e6,
              "gae_frac": gae_b / gae_ms / 1e6 / hbm_, "gather_frac": gat_b / gat_ms / 1e6 / hbm_,
              "frac_of_peak": (gae_b + gat_b) / (gae_ms + gat_ms) / 1e6 / hbm_, "peak_gbs": hbm_,
              "peak_kind": pk,
              "bytes_per_step": {"gae": 17, "gather": 8 * D_ + 36}}
        del v5

    # ---- collection-side inference engine: every env requests
    # each batch; one process_batch = requests H2D, act + sampling, actions D2H,
    # protocol bookkeeping and store appends (wall clock around the C-ABI call)
    coll = None
    if rank == 0 and not args.no_collect:
        NC = 4096
        eng = V.InferenceEngine(cfg, T_, NC, params, version=1, mode=V.VARIABLE, seed=mix(1, 0xC011), ctx=ctx)
        eng.begin_rollout()
        crng = np.random.default_rng(21)
        envc = np.arange(NC, dtype=np.int32)
        stp = np.zeros(NC, np.int32)
        epc = np.zeros(NC, np.int64)
        eng.process_arrays(envc, crng.standard_normal((NC, D_)).astype(np.float32), first=np.ones(NC, np.uint8),
                           obs_episode=epc, obs_step=stp)
        ct = []
        for b in range(40):
            stp += 1
            ob = crng.standard_normal((NC, D_)).astype(np.float32)
            t0 = time.perf_counter()
            eng.process_arrays(envc, ob, reward=np.ones(NC, np.float32), done=np.zeros(NC, np.uint8),
                               obs_episode=epc, obs_step=stp)
            ct.append(time.perf_counter() - t0)
            if eng.rollout_done():
                eng.close()
                eng.begin_rollout()
        cms = 1000.0 * statistics.median(ct[5:])
        coll = {"workload": f"InferenceEngine.process_batch, {NC} envs x 1 step, encoder 2x{E_} + GRU-{H_}, "
                            f"{A_} discrete actions, counter-RNG sampling on device",
                "envs": NC, "ms_per_batch": cms, "actions_per_s": NC / (cms / 1000.0),
                "h2d_bytes_per_batch": NC * (4 * D_ + 4 + 4 + 1 + 1 + 4 + 8 + 4),
                "d2h_bytes_per_batch": NC * (4 + 4)}
        if not args.no_cpu:
            from oracle import engine as OE  # CPU baseline leg only
            NS = 64
            oe = OE.Engine(cfg, T_, NS, params.astype(np.float64), version=1, mode=1, seed=mix(1, 0xC011))
            oe.begin_rollout()
            oe.process_batch([OE.Request(e, crng.standard_normal(D_), first=True) for e in range(NS)])
            t0 = time.perf_counter()
            for b in range(2):
                oe.process_batch([OE.Request(e, crng.standard_normal(D_), reward=1.0, obs_step=b + 1)
                                  for e in range(NS)])
            cdt = time.perf_counter() - t0
            coll["cpu_baseline"] = {"value": 2 * NS / cdt, "unit": "actions/s", "cores": 1, "kind": "port",
                                    "sample": f"oracle engine (double act), {NS} envs x 2 batches ({cdt:.1f} s)"}
        del eng

    # ---- overlapped collection + learning (bench.cpp:129-160): C2
    # iterations (collect one rollout of N envs x T steps through the engine, update on
    # the previous one) serially and with the engine and the learner on separate
    # streams / host threads
    ovl = None
    if rank == 0 and world == 1 and not args.no_collect:
        from paper_2210_05064_b200.overlap import OverlappedTrainer
        ce, cl = V.Context(local), V.Context(local)
        eng2 = V.InferenceEngine(cfg, T_, N2, params, version=0, mode=V.VARIABLE, seed=mix(2, 0xC011), ctx=ce)
        lrn2 = V.Learner(cfg, params, V.PPOConfig(epochs=EPOCHS2, minibatches=MINIBATCHES), V.EntropyController(),
                         V.CosineSchedule(2.5e-4, 2_000_000), mix(3, 0xF00D), ctx=cl)
        orng = np.random.default_rng(33)
        oenv = np.arange(N2, dtype=np.int32)

        def ocollect(e):
            e.begin_rollout()
            st_ = np.zeros(N2, np.int32)
            ep_ = np.zeros(N2, np.int64)
            e.process_arrays(oenv, orng.standard_normal((N2, D_)).astype(np.float32), first=np.ones(N2, np.uint8),
                             obs_episode=ep_, obs_step=st_)
            while not e.rollout_done():
                st_ += 1
                e.process_arrays(oenv, orng.standard_normal((N2, D_)).astype(np.float32),
                                 reward=np.ones(N2, np.float32), done=np.zeros(N2, np.uint8), obs_episode=ep_,
                                 obs_step=st_)
            e.finalize_bootstraps()
            return e.close()

        tr = OverlappedTrainer(eng2, lrn2, ocollect)
        tr.prime()
        tr.iteration(read_stats=False)  # warm-up
        seq_ms, ovl_ms = [], []
        for _ in range(5):
            t0 = time.perf_counter()
            v_ = ocollect(eng2)
            ce.synchronize()
            lrn2.update(v_, read_stats=False)
            cl.synchronize()
            seq_ms.append(1000.0 * (time.perf_counter() - t0))
            t0 = time.perf_counter()
            tr.iteration(read_stats=False)
            ovl_ms.append(1000.0 * (time.perf_counter() - t0))
        ovl = {"workload": f"C2 iteration: collect {N2} envs x {T_} steps through InferenceEngine (synthetic env "
                           f"loop) + one learner update", "serial_ms": statistics.median(seq_ms),
               "overlapped_ms": statistics.median(ovl_ms),
               "env_steps_per_s_overlapped": N2 * T_ / (statistics.median(ovl_ms) / 1000.0)}
        del tr, eng2, lrn2

    if rank == 0:
        hbm, bf16, bf16s, peaks_kind = load_peaks()
        n_mb = EPOCHS * MINIBATCHES
        gemm_ms = phase.get("gemm_fwd", 0.0) + phase.get("gemm_bwd", 0.0)
        rec_ms = phase.get("rec_fwd", 0.0) + phase.get("rec_bwd", 0.0)
        if gemm_ms >= rec_ms:
            # dominant kernel family: the tcgen05 3xTF32 GEMMs (encoder, input projection,
            # backward data / weight gradients); achieved = their algorithmic 2MNK FLOPs
            # (counted per launch by the library) / their device time (CUDA events
            # around each launch on the library stream)
            gflop = flop.get("gemm_fwd", 0.0) + flop.get("gemm_bwd", 0.0)
            n_l = phase_n.get("gemm_fwd", 0) + phase_n.get("gemm_bwd", 0)
            achieved_tf = gflop / (gemm_ms / 1000.0) / 1e12 if gemm_ms > 0 else 0.0
            tr_ = traffic_entry("tc_gemm_c3")
            roof = {"bound": "tensor", "achieved": achieved_tf, "peak": bf16s, "unit": "TFLOP/s",
                    "frac": achieved_tf / bf16s,
                    "traffic": tr_.get("dram_bytes_per_launch") if tr_ else None,
                    "kernel": (f"tc_gemm_kernel (tcgen05 kind::tf32, 3xTF32 fp32-grade): {n_l} launches per update, "
                               f"{gflop / 1e12:.2f} TFLOP algorithmic (2MNK) in {gemm_ms:.2f} ms"),
                    "peak_kind": f"{peaks_kind} bf16 dense sustained (3xTF32 issues 3 tf32 MMAs per product "
                                 f"at half the bf16 rate: its own ceiling is peak/6)",
                    "frac_of_3xtf32_ceiling": achieved_tf / (bf16s / 6.0)}
            if tr_:
                roof["traffic_launch"] = tr_.get("launch")
        else:
            rows_per_mb = fresh * EPOCHS / n_mb
            dom = max(("rec_bwd", "rec_fwd"), key=lambda k: phase.get(k, 0.0))
            dom_ms = phase.get(dom, 0.0) / n_mb
            achieved_tf = 6.0 * H_ * H_ * rows_per_mb / (dom_ms / 1000.0) / 1e12 if dom_ms > 0 else 0.0
            tr_ = traffic_entry("rec_bwd_c3") if dom == "rec_bwd" else None  # (captured at C3: N_ = 4096)
            roof = {"bound": "tensor", "achieved": achieved_tf, "peak": bf16s, "unit": "TFLOP/s",
                    "frac": achieved_tf / bf16s,
                    # DRAM bytes of all backward recurrence launches of one minibatch (the
                    # same unit as `achieved`), from the committed ncu captures
                    "traffic": tr_.get("dram_bytes_per_launch") if tr_ else None,
                    "kernel": f"GRU recurrence {dom}: {dom_ms:.3f} ms per minibatch for {rows_per_mb:.0f} rows x 6H^2",
                    "peak_kind": f"{peaks_kind} bf16 dense sustained",
                    # the backward recurrence issues 3 tf32 MMAs per product (3xTF32) at half
                    # the bf16 rate: its own tensor ceiling is peak / 6
                    "frac_of_3xtf32_ceiling": achieved_tf / (bf16s / 6.0)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic (SURVEY.md §8d generator, random-init policy)",
            "config": {"workload": (f"configs[{2 if world == 1 else 3}]: N={N_} envs/GPU lognormal step times, "
                                    f"T={T_}, encoder 2x{E_} + GRU-{H_}, {EPOCHS} epochs x {MINIBATCHES} minibatches"),
                       "fresh_steps_per_gpu": fresh, "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"dp{world} (DD-PPO, NCCL AllReduce per minibatch)" if world > 1 else "dp1"},
            "roofline": roof,
            "phases_ms": phase,
            "phase_counts": phase_n,
            "gpu_launches": int(launches),
            "step_ms_rank0": [round(x, 3) for x in step_ms],  # each timed step (CUDA events), this rank
            "clocks": clk.summary(),
            "e2e": {"value": fresh * world / (e2e / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8 * 12, "ms_per_step": e2e},
        }
        if lat:
            line["gru_latency"] = lat
        if c2:
            line["c2"] = c2
        if gg:
            line["gae_gather"] = gg
        if coll:
            line["collect"] = coll
        if ovl:
            line["overlap"] = ovl
        if not args.no_cpu and world == 1:
            cv, dt, thr, sample = cpu_sample(2 * args.ref_envs)  # ~10 s of CPU work
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-c2", action="store_true", help="skip the configs[1] (C2) extra field")
    ap.add_argument("--no-c5", action="store_true", help="skip the GAE+gather ragged sweep point")
    ap.add_argument("--no-collect", action="store_true", help="skip the inference-engine measurements")
    ap.add_argument("--c5-log2", type=int, default=26, help="log2 steps of the GAE+gather point")
    ap.add_argument("--ref-envs", type=int, default=128, help="envs of the CPU oracle sample per reference-arm step (the cpu_baseline leg uses 2x)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
