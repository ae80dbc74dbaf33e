"""The C++ host side above the C-ABI (include/ver_gpu.hpp), driven like the
reference's train_single (bench.cpp:95-205).

CPU: the wrapper compiles against include/, links libver_b200.so and maps a
missing device to DeviceError.  GPU: the C++ caller's update equals the Python
API's update on the same records bit for bit (same library, same kernels)."""
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2210_05064_b200" / "_lib"
SRC = ROOT / "tests" / "cpp" / "wrapper_update.cpp"
OUT = ROOT / "tests" / "cpp" / "_build" / "wrapper_update"


def _build():
    OUT.parent.mkdir(parents=True, exist_ok=True)
    if not OUT.exists() or OUT.stat().st_mtime < max(SRC.stat().st_mtime,
                                                     (ROOT / "include" / "ver_gpu.hpp").stat().st_mtime,
                                                     (LIB / "libver_b200.so").stat().st_mtime):
        subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", str(ROOT / "include"), str(SRC),
                        "-L", str(LIB), "-lver_b200", f"-Wl,-rpath,{LIB}", "-o", str(OUT)], check=True)
    return OUT


def _has_gpu():
    return any(Path("/dev").glob("nvidia[0-9]*"))


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device error path")
def test_wrapper_builds_and_maps_device_error():
    exe = _build()
    r = subprocess.run([str(exe), "nodevice"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DeviceError" in r.stdout


@pytest.mark.gpu
def test_wrapper_update_matches_python_api(tmp_path):
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    exe = _build()
    T, N, D, H = 16, 8, 2, 16
    wl = synth.make_workload(T, N, hidden_dim=H, seed=5)
    rec = wl.records
    n = len(rec)
    (tmp_path / "meta.txt").write_text(f"{T} {N} {D} {H} {n}\n")
    hb = np.zeros((n, H), np.float32) if rec.h_before is None else np.asarray(rec.h_before, np.float32)
    hbv = (np.zeros(n, np.uint8) if rec.h_before_valid is None
           else np.asarray(rec.h_before_valid, np.uint8))
    for name, arr in (("env.i32", np.asarray(rec.env_index, np.int32)),
                      ("obs.f32", np.asarray(rec.obs, np.float32)),
                      ("act.i32", np.asarray(rec.act_disc, np.int32)),
                      ("logp.f32", np.asarray(rec.log_prob, np.float32)),
                      ("value.f32", np.asarray(rec.value, np.float32)),
                      ("reward.f32", np.asarray(rec.reward, np.float32)),
                      ("done.u8", np.asarray(rec.done, np.uint8)),
                      ("hb.f32", hb), ("hbv.u8", hbv),
                      ("boot.f32", np.asarray(wl.bootstrap, np.float32)),
                      ("bootv.u8", np.asarray(wl.bootstrap_valid, np.uint8))):
        np.ascontiguousarray(arr).tofile(tmp_path / name)
    cfg = V.ModelConfig(obs_dim=D, encoder_dim=H, hidden_dim=H, action_kind=0, num_actions=2)
    p0 = np.asarray(V.params_init(cfg, 3), np.float32)
    p0.tofile(tmp_path / "params.f32")
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    p_cpp = np.fromfile(tmp_path / "params_out.f32", np.float32)

    buf = V.RolloutBuffer(T, N, V.VARIABLE, 0, D, 0, H)
    synth.fill_buffer(buf, wl)
    view = buf.close_rollout()
    L = V.Learner(cfg, p0, V.PPOConfig(epochs=2, minibatches=2), V.EntropyController(),
                  V.CosineSchedule(2.5e-4, 1_000_000), 77)
    L.update(view)
    p_py = np.asarray(L.params(), np.float32)
    assert p_cpp.shape == p_py.shape
    assert np.array_equal(p_cpp, p_py)
    assert not np.array_equal(p_cpp, p0)


@pytest.mark.gpu
def test_wrapper_engine_matches_python_api(tmp_path):
    """ver::gpu::InferenceEngine (C++) and the Python InferenceEngine dispatch the
    same actions on the same requests (same library, same kernels)."""
    import paper_2210_05064_b200 as V
    exe = _build()
    T, N, D, H, steps = 8, 32, 2, 16, 6
    (tmp_path / "meta.txt").write_text(f"{T} {N} {D} {H} {steps}\n")
    cfg = V.ModelConfig(obs_dim=D, encoder_dim=H, hidden_dim=H, action_kind=0, num_actions=2)
    p = np.asarray(V.params_init(cfg, 4), np.float32)
    p.tofile(tmp_path / "params.f32")
    obs = np.random.default_rng(3).standard_normal((steps + 1, N, D)).astype(np.float32)
    obs.tofile(tmp_path / "obs.f32")
    r = subprocess.run([str(exe), "engine", str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    a_cpp = np.fromfile(tmp_path / "actions.i32", np.int32)
    g = V.InferenceEngine(cfg, T, N, p, version=1, mode=V.VARIABLE, seed=12345)
    g.begin_rollout()
    env = np.arange(N, dtype=np.int32)
    acts = []
    for s in range(steps + 1):
        if g.rollout_done():
            break
        _, _, a = g.process_arrays(env, obs[s], reward=np.full(N, 0.5, np.float32),
                                   done=np.zeros(N, np.uint8), first=np.full(N, 1 if s == 0 else 0, np.uint8),
                                   obs_episode=np.zeros(N, np.int64), obs_step=np.full(N, s, np.int32))
        acts.append(a)
    np.testing.assert_array_equal(a_cpp, np.concatenate(acts))
