#!/usr/bin/env python
"""VER learner hot-path benchmark (BASELINE.json metric: learner env-steps/sec;
GAE+gather HBM GB/s vs peak).

Workload (configs[1]): N=256 envs/GPU with lognormal step times, T=128 VER
rollout (32,768 fresh steps), encoder 2x512 + GRU-512 policy (E=H=512, D=2,
A=2), 4 epochs x 2 minibatches, synthetic data.

A step = one full Learner::update (GAE -> 4 epochs x 2 x (split, pack, gather,
split-tail replay, forward, fused PPO loss, backward, [NCCL AllReduce], Adam,
alpha)) on a device-resident closed view.  `e2e` = the same through the C-ABI
with host buffers: append the host arrival log, close_rollout (H2D + device
compaction), update, read the stats back.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

T_, N_, E_, H_, D_, A_ = 128, 256, 512, 512, 2, 2
EPOCHS, MINIBATCHES = 4, 2
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


def dom_traffic(dom):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed `ncu --set full` capture (profiles/traffic.json), or None."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    # one minibatch of one direction = one K-split launch + one persistent step-kernel
    # launch (the cluster tail moves a few MB); both captured from the same update
    ks = d.get("gru_bwd_ks" if dom == "rec_bwd" else "gru_fwd_ks", {}).get("dram_bytes_per_launch")
    sg = d.get("gru_step_gemm_bwd" if dom == "rec_bwd" else "gru_step_gemm_fwd", {}).get("dram_bytes_per_launch")
    if ks is None:
        return None
    return ks + (sg or 0.0)


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
def cpu_sample(n_envs_sample=64, seed=1):
    """The oracle (CPU double restatement, single thread as the reference's
    learner thread) on a bounded sample: N=64 of the 256 envs (same T, model,
    epochs, B), GAE + minibatch 0 of epoch 0 timed, extrapolated to the full
    4 x 2 minibatch update.  Returns (env-steps/s, seconds measured, sample)."""
    from oracle import oracle as O
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    cfg = V.ModelConfig(obs_dim=D_, encoder_dim=E_, hidden_dim=H_, action_kind=0, num_actions=A_)
    wl = synth.make_workload(T_, n_envs_sample, hidden_dim=H_, seed=seed)
    r = O.Rollout(T_, n_envs_sample, 1, 0, D_, 0, H_)
    synth.fill_buffer(r, wl)
    view = r.close_rollout()
    p = O.params_init(cfg, O.mix(seed, 0x9A9A))
    L = O.Learner(cfg, p, V.PPOConfig(epochs=EPOCHS, minibatches=MINIBATCHES), V.EntropyController(),
                  2.5e-4, 2_000_000, O.mix(seed, 0xF00D))
    t0 = time.perf_counter()
    L.update(view, max_minibatches=1)
    dt = time.perf_counter() - t0
    per_update = dt * EPOCHS * MINIBATCHES  # GAE is O(N S) but tiny next to a minibatch
    steps = T_ * n_envs_sample
    return steps / per_update, dt, (f"oracle port, 1 thread: N={n_envs_sample} of {N_} envs, T={T_}, "
                                    f"E=H={E_}, GAE + 1 of {EPOCHS}x{MINIBATCHES} minibatches timed "
                                    f"({dt:.1f} s), extrapolated x{EPOCHS * MINIBATCHES}")


def run_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample()
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, dt, sample = cpu_sample()
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * wall / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8d generator)",
        "config": {"workload": f"configs[1]: N={N_} envs, T={T_}, encoder 2x{E_} + GRU-{H_}, "
                               f"{EPOCHS} epochs x {MINIBATCHES} minibatches (sampled, see cpu_baseline)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU side
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
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        ctx.synchronize()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    # ---- device-resident learner updates
    for _ in range(args.warmup):
        learner.update(view, read_stats=False)
    barrier()
    n0 = ctx.launch_count()
    times = []
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # L2 flush between timed steps (outside the event pair)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            learner.update(view, read_stats=False)
            with torch.cuda.stream(stream):
                e1.record(stream)
            times.append((e0, e1))
        barrier()
    launches = (ctx.launch_count() - n0) // max(1, args.steps)
    step_ms = [a.elapsed_time(b) for a, b in times]
    ms = sum(step_ms) / len(step_ms)
    phase = learner.last_timing()
    phase_n = learner.last_timing_counts()
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = fresh * world / (ms / 1000.0)

    # ---- e2e through the C-ABI with host buffers
    e2e_ms = []
    rec = wl.records
    h2d = sum(np.asarray(getattr(rec, f)).nbytes for f in ("env_index", "obs", "log_prob", "value", "reward",
                                                           "done", "act_disc", "episode_index",
                                                           "step_in_episode", "latency", "snapshot_version"))
    h2d += 4 * 3 * len(rec)  # env rank / h-slot / rank columns of the arrival log
    h2d += N_ * (H_ * 4 + 9)  # h0 rows of rollout-start sequences (upper bound) + bootstrap
    for i in range(max(1, args.steps)):
        barrier()
        t0 = time.perf_counter()
        synth.fill_buffer(buf, wl, snapshot_version=2 + i)
        v2 = buf.close_rollout()
        st = learner.update(v2)
        barrier()
        e2e_ms.append(1000.0 * (time.perf_counter() - t0))
        del v2
    e2e = statistics.median(e2e_ms)
    if dist:
        t = torch.tensor([e2e], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())

    # ---- GAE + gather HBM throughput on the ragged stress view
    gg = None
    if rank == 0 and not args.no_c5:
        S5 = 1 << args.c5_log2
        lens = synth.ragged_lengths(S5, seed=11)
        v5 = V.view_synth(lens, obs_dim=D_, hidden_dim=4, seed=12, ctx=ctx)
        gae_ms, gat_ms = V.bench_gae_gather(v5, B=MINIBATCHES, seed=13, reps=5)
        hbm_, _, _, pk = load_peaks()
        gae_b = 17.0 * S5 + 9.0 * len(lens)          # r, V, done in; A, R out; + bootstrap/valid/offset per env
        gat_b = (8.0 * D_ + 36.0) * S5               # obs, act, old log-prob, A, R in + out, slot out
        gg = {"steps": S5, "envs": int(len(lens)), "gae_ms": gae_ms, "gather_ms": gat_ms,
              "gae_gbs": gae_b / gae_ms / 1e6, "gather_gbs": gat_b / gat_ms / 1e6,
              "gae_gather_gbs": (gae_b + gat_b) / (gae_ms + gat_ms) / 1e6,
              "frac_of_peak": (gae_b + gat_b) / (gae_ms + gat_ms) / 1e6 / hbm_, "peak_gbs": hbm_,
              "peak_kind": pk,
              "bytes_per_step": {"gae": 17, "gather": 8 * D_ + 36}}
        del v5

    # ---- C3 (configs[2]): N = 4096 envs, GRU-512, 3 epochs (reference default) x 2 minibatches
    c3 = None
    if rank == 0 and not args.no_c3:
        N3, EP3 = 4096, 3
        wl3 = synth.make_workload(T_, N3, obs_dim=D_, num_actions=A_, hidden_dim=H_, seed=3)
        buf3 = V.RolloutBuffer(T_, N3, V.VARIABLE, 0, D_, 0, H_, ctx=ctx)
        synth.fill_buffer(buf3, wl3)
        view3 = buf3.close_rollout()
        l3 = V.Learner(cfg, params, V.PPOConfig(epochs=EP3, minibatches=MINIBATCHES), V.EntropyController(),
                       V.CosineSchedule(2.5e-4, 2_000_000), mix(3, 0xF00D), ctx=ctx)
        l3.update(view3, read_stats=False)
        barrier()
        t3 = []
        for _ in range(2):
            with torch.cuda.stream(stream):
                flush.fill_(1)
                a_ = torch.cuda.Event(enable_timing=True)
                b_ = torch.cuda.Event(enable_timing=True)
                a_.record(stream)
            l3.update(view3, read_stats=False)
            with torch.cuda.stream(stream):
                b_.record(stream)
            t3.append((a_, b_))
        barrier()
        ms3 = sum(a_.elapsed_time(b_) for a_, b_ in t3) / len(t3)
        f3 = view3.fresh_steps()
        c3 = {"workload": f"configs[2]: N={N3} envs, T={T_}, encoder 2x{E_} + GRU-{H_}, {EP3} epochs x "
                          f"{MINIBATCHES} minibatches", "fresh_steps": f3, "ms_per_update": ms3,
              "env_steps_per_s": f3 / (ms3 / 1000.0), "phases_ms": l3.last_timing()}
        del l3, view3, buf3

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
        eng2 = V.InferenceEngine(cfg, T_, N_, params, version=0, mode=V.VARIABLE, seed=mix(2, 0xC011), ctx=ce)
        lrn2 = V.Learner(cfg, params, V.PPOConfig(epochs=EPOCHS, minibatches=MINIBATCHES), V.EntropyController(),
                         V.CosineSchedule(2.5e-4, 2_000_000), mix(3, 0xF00D), ctx=cl)
        orng = np.random.default_rng(33)
        oenv = np.arange(N_, dtype=np.int32)

        def ocollect(e):
            e.begin_rollout()
            st_ = np.zeros(N_, np.int32)
            ep_ = np.zeros(N_, np.int64)
            e.process_arrays(oenv, orng.standard_normal((N_, D_)).astype(np.float32), first=np.ones(N_, np.uint8),
                             obs_episode=ep_, obs_step=st_)
            while not e.rollout_done():
                st_ += 1
                e.process_arrays(oenv, orng.standard_normal((N_, D_)).astype(np.float32),
                                 reward=np.ones(N_, np.float32), done=np.zeros(N_, np.uint8), obs_episode=ep_,
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
        ovl = {"workload": f"C2 iteration: collect {N_} envs x {T_} steps through InferenceEngine (synthetic env "
                           f"loop) + one learner update", "serial_ms": statistics.median(seq_ms),
               "overlapped_ms": statistics.median(ovl_ms),
               "env_steps_per_s_overlapped": fresh / (statistics.median(ovl_ms) / 1000.0)}
        del tr, eng2, lrn2

    if rank == 0:
        hbm, bf16, bf16s, peaks_kind = load_peaks()
        # dominant kernel = the GRU recurrence direction with the larger device time
        # (the launch list in profiles/ ranks it first): per minibatch one K-split
        # launch (+ one cluster-tail launch); its algorithmic work is one H x 3H
        # matvec per packed row (6 H^2 FLOP), every row once per epoch
        dom = max(("rec_bwd", "rec_fwd"), key=lambda k: phase.get(k, 0.0))
        n_mb = EPOCHS * MINIBATCHES
        n_dom = max(1, phase_n.get(dom, 0))
        rows_per_mb = fresh * EPOCHS / n_mb
        dom_flop = 6.0 * H_ * H_ * rows_per_mb
        dom_ms = phase.get(dom, 0.0) / n_mb
        achieved_tf = dom_flop / (dom_ms / 1000.0) / 1e12 if dom_ms > 0 else 0.0
        simt_peak = 148 * 128 * 2 * 1.965e9 / 1e12  # fp32 FMA pipe peak at max SM clock
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic (SURVEY.md §8d generator, seed 1)",
            "config": {"workload": f"configs[1]: N={N_} envs/GPU lognormal step times, T={T_}, encoder 2x{E_}"
                                   f" + GRU-{H_}, {EPOCHS} epochs x {MINIBATCHES} minibatches",
                       "fresh_steps_per_gpu": fresh, "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"dp{world} (DD-PPO, NCCL AllReduce per minibatch)" if world > 1 else "dp1"},
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": bf16s, "unit": "TFLOP/s",
                         "frac": achieved_tf / bf16s, "traffic": dom_traffic(dom),
                         "kernel": (f"{'gru_step_gemm_kernel<1> + gru_bwd_ks<512> + gru_bwd_tail<512>' if dom == 'rec_bwd' else 'gru_step_gemm_kernel<0> + gru_fwd_ks<512> + gru_fwd_tail<512>'}"
                                    f" (GRU recurrence: tcgen05 3xTF32 steps >= 150 rows, fp32 FMA pipe below; {n_dom} launches/step over {n_mb} minibatches, "
                                    f"{dom_ms:.3f} ms per minibatch for {rows_per_mb:.0f} rows x 6H^2 FLOP)"),
                         "peak_kind": f"{peaks_kind} bf16 dense sustained",
                         "fp32_simt_peak": simt_peak, "frac_of_fp32_simt": achieved_tf / simt_peak},
            "phases_ms": phase,
            "phase_counts": phase_n,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "e2e": {"value": fresh * world / (e2e / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": 8 * 12, "ms_per_step": e2e},
        }
        if gg:
            line["gae_gather"] = gg
        if c3:
            line["c3"] = c3
        if coll:
            line["collect"] = coll
        if ovl:
            line["overlap"] = ovl
        if not args.no_cpu and world == 1:
            cv, dt, sample = cpu_sample()
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
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
    ap.add_argument("--no-c5", action="store_true", help="skip the GAE+gather ragged sweep point")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 (N=4096) update measurement")
    ap.add_argument("--no-collect", action="store_true", help="skip the inference-engine measurement")
    ap.add_argument("--c5-log2", type=int, default=26, help="log2 steps of the GAE+gather point")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
