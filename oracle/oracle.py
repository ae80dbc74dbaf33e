"""ctypes binding of the CPU double-precision oracle (oracle/ver_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, always as the checker or
the timed CPU baseline, never as a product path.

Parity status: the oracle restates /root/reference/proj line by line (the
reference itself needs Eigen3/doctest/CLI11, absent here) and is pinned by
ports of every known-answer and property test the reference holds for the
hot path (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libver_oracle.so"

P = C.POINTER
c_int, c_int32, c_int64, c_uint64, c_double = C.c_int, C.c_int32, C.c_int64, C.c_uint64, C.c_double


class ViewData(C.Structure):
    _fields_ = [
        ("T", c_int), ("N", c_int), ("action_kind", c_int), ("obs_dim", c_int), ("act_dim", c_int),
        ("hidden_dim", c_int), ("size", c_int), ("num_seqs", c_int), ("deficit", c_int),
        ("stale_steps", c_int), ("replayed_steps", c_int), ("snapshot_version", c_uint64),
        ("collect_wall_time", c_double),
        ("obs", P(c_double)), ("act_cont", P(c_double)), ("act_disc", P(c_int32)),
        ("log_prob", P(c_double)), ("value", P(c_double)), ("reward", P(c_double)),
        ("latency", P(c_double)), ("advantage", P(c_double)), ("returns", P(c_double)),
        ("done", P(C.c_uint8)), ("stale", P(C.c_uint8)), ("replayed", P(C.c_uint8)),
        ("env_index", P(c_int32)), ("seq_of_slot", P(c_int32)), ("step_in_episode", P(c_int32)),
        ("episode_index", P(c_int64)), ("version", P(c_uint64)),
        ("seqs", P(c_int32)), ("h0", P(c_double)), ("h0_rows", c_int),
        ("per_env_counts", P(c_int32)), ("env_bootstrap", P(c_double)),
        ("env_bootstrap_valid", P(C.c_uint8)),
    ]


class ModelCfg(C.Structure):
    _fields_ = [("obs_dim", c_int), ("encoder_dim", c_int), ("hidden_dim", c_int),
                ("action_kind", c_int), ("num_actions", c_int), ("act_dim", c_int)]


class PPOCfg(C.Structure):
    _fields_ = [("gamma", c_double), ("gae_lambda", c_double), ("clip", c_double), ("epochs", c_int),
                ("minibatches", c_int), ("value_loss_coef", c_double), ("is_cap", c_double)]


class LossRes(C.Structure):
    _fields_ = [(n, c_double) for n in ("loss", "policy_loss", "value_loss", "mean_entropy",
                                         "ratio_sum", "clip_count", "w_sum", "w_max")] + [("steps", c_int)]


class EntCtl(C.Structure):
    _fields_ = [(n, c_double) for n in ("alpha", "target", "lower", "upper", "lr")]


class Stats(C.Structure):
    _fields_ = [("update_index", c_int64), ("steps", c_int), ("fresh_steps", c_int),
                ("stale_steps", c_int)] + [
        (n, c_double) for n in ("loss", "policy_loss", "value_loss", "entropy", "entropy_loss",
                                "mean_ratio", "clip_fraction", "mean_is_weight", "max_is_weight",
                                "alpha", "lr")]


GRAD_HOOK = C.CFUNCTYPE(None, P(c_double), c_int64, C.c_void_p)
ENT_HOOK = C.CFUNCTYPE(c_double, c_double, C.c_void_p)


class OracleProtocolError(RuntimeError):
    pass


class OracleConfigError(RuntimeError):
    pass


_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.vo_last_error.restype = C.c_char_p
        L.vo_mix.restype = c_uint64
        L.vo_mix.argtypes = [c_uint64, c_uint64]
        L.vo_splitmix64.restype = c_uint64
        L.vo_splitmix64.argtypes = [c_uint64]
        L.vo_cosine_lr.restype = c_double
        L.vo_cosine_lr.argtypes = [c_double, c_int64, c_int64]
        L.vo_categorical_log_prob.restype = c_double
        L.vo_categorical_log_prob.argtypes = [P(c_double), c_int, c_int]
        L.vo_categorical_entropy.restype = c_double
        L.vo_categorical_entropy.argtypes = [P(c_double), c_int]
        L.vo_merged_time.restype = c_double
        L.vo_merged_time.argtypes = [P(c_double), c_int, c_int64]
        L.vo_entropy_update.restype = c_double
        L.vo_entropy_update.argtypes = [P(EntCtl), c_double]
        L.vo_estimate_time.argtypes = [P(c_double), c_int, c_int64, c_int64, P(c_double)]
        L.vo_optimal_preempt_steps.argtypes = [P(c_double), c_int, c_double, c_int64, P(c_int64)]
        L.vo_optimal_preempt_steps_sorted.argtypes = [P(c_double), c_int, c_double, c_int64, P(c_int64)]
        L.vo_rollout_begin.argtypes = [C.c_void_p, c_uint64]
        L.vo_split_minibatches.argtypes = [C.c_void_p, c_int, c_uint64, P(C.c_void_p)]
        L.vo_shuffle_perm.argtypes = [c_int, c_uint64, P(c_int32)]
        L.vo_params_init.argtypes = [P(ModelCfg), c_uint64, P(c_double)]
        L.vo_ppo_loss.argtypes = [P(ModelCfg), P(c_double), C.c_void_p, C.c_void_p, P(PPOCfg), c_double,
                                  P(c_double), c_int, P(c_double), P(LossRes), P(c_double), P(c_double)]
        L.vo_learner_create.argtypes = [P(ModelCfg), P(c_double), P(PPOCfg), P(EntCtl), c_double,
                                        c_int64, c_uint64, P(C.c_void_p)]
        L.vo_learner_set_hooks.argtypes = [C.c_void_p, GRAD_HOOK, ENT_HOOK, C.c_void_p]
        L.vo_learner_set_state.argtypes = [C.c_void_p, c_double, c_int64, c_int64]
        L.vo_adam_step.argtypes = [c_int64, P(c_double), P(c_double), P(c_double), P(c_double),
                                   P(c_int64), c_double]
        L.vo_view_restale.argtypes = [C.c_void_p, c_uint64]
        for fn in ("vo_view_destroy", "vo_rollout_destroy", "vo_groups_destroy", "vo_packed_destroy",
                   "vo_learner_destroy"):
            getattr(L, fn).argtypes = [C.c_void_p]
            getattr(L, fn).restype = None
        L.vo_set_num_threads.argtypes = [c_int]
        # threads of the oracle's GEMMs / reductions: results are bit-identical for
        # any count; VER_ORACLE_THREADS (tests: all cores) or 1 (the reference's
        # single learner thread)
        import os
        L.vo_set_num_threads(int(os.environ.get("VER_ORACLE_THREADS", "1")))
        L.vo_set_sparse_rows.argtypes = [c_int]
        L.vo_set_sparse_rows(int(os.environ.get("VER_ORACLE_SPARSE_ROWS", "0")))
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle (bit-identical results for any count)."""
    lib().vo_set_num_threads(int(n))


def set_sparse_rows(on: bool) -> None:
    """`rows` backward without the full-size scatter temporary (identical sums)."""
    lib().vo_set_sparse_rows(int(on))


def get_threads() -> int:
    return int(lib().vo_get_num_threads())


def _chk(r: int):
    if r == 0:
        return
    msg = lib().vo_last_error().decode()
    if r == 1:
        raise OracleProtocolError(msg)
    raise OracleConfigError(msg)


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(P(ct))


def mix(a: int, b: int) -> int:
    return lib().vo_mix(a, b)


# ------------------------------------------------------------------ views
def _vd_from(hv) -> tuple[ViewData, list]:
    from paper_2210_05064_b200.hostview import HostView  # plain data container
    h: HostView = hv.astype(np.float64)
    d = ViewData()
    d.T, d.N, d.action_kind, d.obs_dim, d.act_dim, d.hidden_dim = (
        h.T, h.N, h.action_kind, h.obs_dim, h.act_dim, h.hidden_dim)
    d.size, d.num_seqs, d.h0_rows = h.size, h.num_seqs, h.h0.shape[0]
    d.deficit, d.stale_steps, d.replayed_steps = h.deficit, h.stale_steps, h.replayed_steps
    d.snapshot_version, d.collect_wall_time = h.snapshot_version, h.collect_wall_time
    for name, ct in (("obs", c_double), ("act_cont", c_double), ("act_disc", c_int32),
                     ("log_prob", c_double), ("value", c_double), ("reward", c_double),
                     ("latency", c_double), ("advantage", c_double), ("returns", c_double),
                     ("done", C.c_uint8), ("stale", C.c_uint8), ("replayed", C.c_uint8),
                     ("env_index", c_int32), ("seq_of_slot", c_int32), ("step_in_episode", c_int32),
                     ("episode_index", c_int64), ("version", c_uint64), ("seqs", c_int32),
                     ("h0", c_double), ("per_env_counts", c_int32), ("env_bootstrap", c_double),
                     ("env_bootstrap_valid", C.c_uint8)):
        a = getattr(h, name)
        setattr(d, name, _p(a, ct) if a.size else None)
    return d, [h]


class View:
    def __init__(self, h):
        self.h = h

    @staticmethod
    def from_host(hv) -> "View":
        d, keep = _vd_from(hv)
        out = C.c_void_p()
        _chk(lib().vo_view_create(C.byref(d), C.byref(out)))
        return View(out)

    def __del__(self):
        try:
            if self.h:
                lib().vo_view_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def to_host(self):
        from paper_2210_05064_b200.hostview import HostView
        d = ViewData()
        _chk(lib().vo_view_info(self.h, C.byref(d)))
        hv = HostView.empty(d.T, d.N, d.action_kind, d.obs_dim, d.act_dim, d.hidden_dim, d.size,
                            d.num_seqs, d.h0_rows, fdtype=np.float64)
        hv.deficit, hv.stale_steps, hv.replayed_steps = d.deficit, d.stale_steps, d.replayed_steps
        hv.snapshot_version, hv.collect_wall_time = d.snapshot_version, d.collect_wall_time
        d2, _ = _vd_from(hv)  # float64 already: astype copies, so re-point at hv arrays
        for name, ct in (("obs", c_double), ("act_cont", c_double), ("act_disc", c_int32),
                         ("log_prob", c_double), ("value", c_double), ("reward", c_double),
                         ("latency", c_double), ("advantage", c_double), ("returns", c_double),
                         ("done", C.c_uint8), ("stale", C.c_uint8), ("replayed", C.c_uint8),
                         ("env_index", c_int32), ("seq_of_slot", c_int32),
                         ("step_in_episode", c_int32), ("episode_index", c_int64),
                         ("version", c_uint64), ("seqs", c_int32), ("h0", c_double),
                         ("per_env_counts", c_int32), ("env_bootstrap", c_double),
                         ("env_bootstrap_valid", C.c_uint8)):
            a = getattr(hv, name)
            setattr(d2, name, _p(a, ct) if a.size else None)
        if hv.action_kind == 0:
            d2.act_cont = None
        else:
            d2.act_disc = None
        _chk(lib().vo_view_read(self.h, C.byref(d2)))
        return hv

    def clone(self) -> "View":
        out = C.c_void_p()
        _chk(lib().vo_view_clone(self.h, C.byref(out)))
        return View(out)

    def restale(self, lv: int):
        _chk(lib().vo_view_restale(self.h, lv))


class Rollout:
    def __init__(self, T, N, mode=1, action_kind=0, obs_dim=1, act_dim=0, hidden_dim=0):
        self.h = C.c_void_p()
        self.obs_dim, self.act_dim, self.hidden_dim, self.action_kind = obs_dim, act_dim, hidden_dim, action_kind
        _chk(lib().vo_rollout_create(T, N, mode, action_kind, obs_dim, act_dim, hidden_dim, C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                lib().vo_rollout_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def begin_rollout(self, sv: int):
        _chk(lib().vo_rollout_begin(self.h, sv))

    def append_steps(self, recs) -> np.ndarray:
        """recs: paper_2210_05064_b200.api.StepRecords-like (float arrays upcast to double)."""
        n = len(recs)
        keep = []

        def arr(x, dt):
            if x is None:
                return None
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a

        out = np.zeros(n, np.int32)
        _chk(lib().vo_rollout_append_batch(
            self.h, n, _p(arr(recs.env_index, np.int32), c_int32),
            _p(arr(recs.episode_index, np.int64), c_int64),
            _p(arr(recs.step_in_episode, np.int32), c_int32), _p(arr(recs.obs, np.float64), c_double),
            _p(arr(recs.act_disc, np.int32), c_int32), _p(arr(recs.act_cont, np.float64), c_double),
            _p(arr(recs.log_prob, np.float64), c_double), _p(arr(recs.value, np.float64), c_double),
            _p(arr(recs.reward, np.float64), c_double), _p(arr(recs.done, np.uint8), C.c_uint8),
            _p(arr(recs.latency, np.float64), c_double), _p(arr(recs.h_before, np.float64), c_double),
            _p(arr(recs.h_before_valid, np.uint8), C.c_uint8),
            _p(arr(recs.snapshot_version, np.uint64), c_uint64), _p(out, c_int32)))
        return out

    def force_close(self):
        _chk(lib().vo_rollout_force_close(self.h))

    def set_bootstrap(self, env: int, value: float):
        _chk(lib().vo_rollout_set_bootstrap(self.h, env, c_double(value)))

    def state(self):
        o, c, k = c_int(), c_int(), c_int()
        _chk(lib().vo_rollout_state(self.h, C.byref(o), C.byref(c), C.byref(k)))
        return o.value, c.value, k.value

    def close_rollout(self) -> View:
        out = C.c_void_p()
        _chk(lib().vo_rollout_close(self.h, C.byref(out)))
        return View(out)


def backfill_stale(view: View, prev: View, deficit: int):
    _chk(lib().vo_backfill_stale(view.h, prev.h, deficit))


def compute_gae(view: View, gamma: float, lam: float):
    _chk(lib().vo_compute_gae(view.h, c_double(gamma), c_double(lam)))


def gae_arrays(reward, value, done, env, replayed, N, boot, boot_valid, gamma, lam, reference_loop=False):
    """compute_gae (learner.cpp:11-41) over SoA arrays (the C5 CPU baseline):
    reference_loop = the reference's O(N S) slot search, else an O(S) bucketing
    pass before the same per-env recursion.  Returns (advantage, returns)."""
    r = np.ascontiguousarray(reward, np.float32)
    S = r.size
    v = np.ascontiguousarray(value, np.float32)
    d = np.ascontiguousarray(done, np.uint8)
    e = np.ascontiguousarray(env, np.int32)
    rp = np.ascontiguousarray(replayed, np.uint8)
    b = np.ascontiguousarray(boot, np.float32)
    bv = np.ascontiguousarray(boot_valid, np.uint8)
    adv = np.zeros(S, np.float32)
    ret = np.zeros(S, np.float32)
    _chk(lib().vo_gae_arrays(_p(r, C.c_float), _p(v, C.c_float), _p(d, C.c_uint8), _p(e, c_int32),
                             _p(rp, C.c_uint8), S, int(N), _p(b, C.c_float), _p(bv, C.c_uint8), c_double(gamma),
                             c_double(lam), 1 if reference_loop else 0, _p(adv, C.c_float), _p(ret, C.c_float)))
    return adv, ret


def shuffle_perm(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.int32)
    _chk(lib().vo_shuffle_perm(n, seed, _p(out, c_int32)))
    return out


class Groups:
    def __init__(self, h):
        self.h = h
        B = c_int()
        _chk(lib().vo_groups_count(h, C.byref(B)))
        self.B = B.value

    def __del__(self):
        try:
            if self.h:
                lib().vo_groups_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def group(self, b: int) -> tuple[np.ndarray, int]:
        n, tot = c_int(), c_int()
        _chk(lib().vo_groups_get(self.h, b, C.byref(n), C.byref(tot), None))
        a = np.zeros((n.value, 8), np.int32)
        _chk(lib().vo_groups_get(self.h, b, None, None, _p(a, c_int32)))
        return a, tot.value

    def groups(self) -> list[tuple[np.ndarray, int]]:
        return [self.group(b) for b in range(self.B)]


def split_minibatches(view: View, B: int, seed: int) -> Groups:
    out = C.c_void_p()
    _chk(lib().vo_split_minibatches(view.h, B, seed, C.byref(out)))
    return Groups(out)


def split_in_order(view: View, B: int, order) -> Groups:
    o = np.ascontiguousarray(order, dtype=np.int32)
    out = C.c_void_p()
    _chk(lib().vo_split_in_order(view.h, B, _p(o, c_int32), o.size, C.byref(out)))
    return Groups(out)


class Packed:
    def __init__(self, seqs):
        s = np.ascontiguousarray(np.asarray(seqs, np.int32).reshape(-1, 8))
        self.h = C.c_void_p()
        _chk(lib().vo_pack(_p(s, c_int32) if s.size else None, s.shape[0], C.byref(self.h)))
        k, L, S = c_int(), c_int(), c_int()
        _chk(lib().vo_packed_info(self.h, C.byref(k), C.byref(L), C.byref(S)))
        self.num_seqs, self.max_len, self.total_steps = k.value, L.value, S.value
        self.seqs = np.zeros((self.num_seqs, 8), np.int32)
        self.sorted_to_group = np.zeros(self.num_seqs, np.int32)
        self.batch_sizes = np.zeros(self.max_len, np.int32)
        self.offsets = np.zeros(self.max_len, np.int32)
        self.slots = np.zeros(self.total_steps, np.int32)
        _chk(lib().vo_packed_get(self.h, _p(self.seqs, c_int32), _p(self.sorted_to_group, c_int32),
                                 _p(self.batch_sizes, c_int32), _p(self.offsets, c_int32),
                                 _p(self.slots, c_int32)))

    def __del__(self):
        try:
            if self.h:
                lib().vo_packed_destroy(self.h)
                self.h = None
        except Exception:
            pass


def pack(seqs) -> Packed:
    return Packed(seqs)


# ------------------------------------------------------------------ model
def _mc(cfg) -> ModelCfg:
    return ModelCfg(cfg.obs_dim, cfg.encoder_dim, cfg.hidden_dim, cfg.action_kind, cfg.num_actions,
                    cfg.act_dim)


def _pc(ppo) -> PPOCfg:
    return PPOCfg(ppo.gamma, ppo.gae_lambda, ppo.clip, ppo.epochs, ppo.minibatches,
                  ppo.value_loss_coef, ppo.is_cap)


def param_count(cfg) -> int:
    n = c_int64()
    _chk(lib().vo_param_count(C.byref(_mc(cfg)), C.byref(n), None))
    return n.value


def params_init(cfg, seed: int) -> np.ndarray:
    out = np.zeros(param_count(cfg), np.float64)
    _chk(lib().vo_params_init(C.byref(_mc(cfg)), seed, _p(out, c_double)))
    return out


def act(cfg, params, obs, h):
    obs = np.ascontiguousarray(obs, np.float64).reshape(-1, cfg.obs_dim)
    h = np.ascontiguousarray(h, np.float64).reshape(-1, cfg.hidden_dim)
    n = obs.shape[0]
    A = cfg.num_actions if cfg.action_kind == 0 else cfg.act_dim
    dist = np.zeros((n, A))
    val = np.zeros(n)
    hn = np.zeros((n, cfg.hidden_dim))
    p = np.ascontiguousarray(params, np.float64)
    _chk(lib().vo_act(C.byref(_mc(cfg)), _p(p, c_double), n, _p(obs, c_double), _p(h, c_double),
                      _p(dist, c_double), _p(val, c_double), _p(hn, c_double)))
    return dist, val, hn


def forward_packed(cfg, params, obs, act_disc, act_cont, batch_sizes, offsets, h0):
    obs = np.ascontiguousarray(obs, np.float64).reshape(-1, cfg.obs_dim)
    S = obs.shape[0]
    bs = np.ascontiguousarray(batch_sizes, np.int32)
    of = np.ascontiguousarray(offsets, np.int32)
    h0 = np.ascontiguousarray(h0, np.float64).reshape(-1, cfg.hidden_dim)
    ad = None if act_disc is None else np.ascontiguousarray(act_disc, np.int32)
    ac = None if act_cont is None else np.ascontiguousarray(act_cont, np.float64)
    lp, en, va = np.zeros(S), np.zeros(S), np.zeros(S)
    p = np.ascontiguousarray(params, np.float64)
    _chk(lib().vo_forward_packed(C.byref(_mc(cfg)), _p(p, c_double), S, _p(obs, c_double), _p(ad, c_int32),
                                 _p(ac, c_double), bs.size, _p(bs, c_int32), _p(of, c_int32),
                                 _p(h0, c_double), h0.shape[0], _p(lp, c_double), _p(en, c_double),
                                 _p(va, c_double)))
    return lp, en, va


def categorical_log_prob(logits, a: int) -> float:
    l = np.ascontiguousarray(logits, np.float64)
    return lib().vo_categorical_log_prob(_p(l, c_double), l.size, a)


def categorical_entropy(logits) -> float:
    l = np.ascontiguousarray(logits, np.float64)
    return lib().vo_categorical_entropy(_p(l, c_double), l.size)


def ppo_loss(cfg, params, view: View, packed: Packed, ppo, alpha, h0_sorted, want_grads=True,
             frozen_w=None):
    p = np.ascontiguousarray(params, np.float64)
    h0 = np.ascontiguousarray(h0_sorted, np.float64)
    fw = None if frozen_w is None else np.ascontiguousarray(frozen_w, np.float64).reshape(-1)
    res = LossRes()
    grads = np.zeros(p.size) if want_grads else None
    isw = np.zeros(packed.total_steps)
    _chk(lib().vo_ppo_loss(C.byref(_mc(cfg)), _p(p, c_double), view.h, packed.h, C.byref(_pc(ppo)),
                           c_double(alpha), _p(h0, c_double), int(want_grads), _p(fw, c_double),
                           C.byref(res), _p(grads, c_double), _p(isw, c_double)))
    out = {f: getattr(res, f) for f, _ in LossRes._fields_}
    out["grads"] = grads
    out["is_weights"] = isw
    return out


class Learner:
    def __init__(self, cfg, params, ppo, entropy, base_lr: float, total_steps: int, run_seed: int):
        self.cfg = cfg
        self.h = C.c_void_p()
        p = np.ascontiguousarray(params, np.float64)
        ec = EntCtl(entropy.alpha, entropy.target, entropy.lower, entropy.upper, entropy.lr)
        _chk(lib().vo_learner_create(C.byref(_mc(cfg)), _p(p, c_double), C.byref(_pc(ppo)), C.byref(ec),
                                     base_lr, total_steps, run_seed, C.byref(self.h)))
        self.P = p.size
        self._hooks = None

    def __del__(self):
        try:
            if self.h:
                lib().vo_learner_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def set_hooks(self, grad_hook, entropy_hook):
        """grad_hook(np.ndarray view of the flat grads) in place; entropy_hook(h) -> h."""
        def g(ptr, n, user):
            arr = np.ctypeslib.as_array(ptr, shape=(n,))
            grad_hook(arr)

        def e(h, user):
            return float(entropy_hook(h))

        self._hooks = (GRAD_HOOK(g), ENT_HOOK(e))
        _chk(lib().vo_learner_set_hooks(self.h, self._hooks[0], self._hooks[1], None))

    def update(self, view: View, max_minibatches: int = -1) -> dict:
        s = Stats()
        if max_minibatches < 0:
            _chk(lib().vo_learner_update(self.h, view.h, C.byref(s)))
        else:
            _chk(lib().vo_learner_update_partial(self.h, view.h, max_minibatches, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def batch_h0(self, view: View, packed: Packed) -> np.ndarray:
        out = np.zeros((packed.num_seqs, self.cfg.hidden_dim))
        _chk(lib().vo_learner_batch_h0(self.h, view.h, packed.h, _p(out, c_double)))
        return out

    def params(self) -> np.ndarray:
        out = np.zeros(self.P)
        _chk(lib().vo_learner_get_params(self.h, _p(out, c_double)))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, np.float64)
        _chk(lib().vo_learner_set_params(self.h, _p(p, c_double)))

    def adam(self):
        m, v, s = np.zeros(self.P), np.zeros(self.P), c_int64()
        _chk(lib().vo_learner_get_adam(self.h, _p(m, c_double), _p(v, c_double), C.byref(s)))
        return m, v, s.value

    def state(self):
        a, c, u = c_double(), c_int64(), c_int64()
        _chk(lib().vo_learner_get_state(self.h, C.byref(a), C.byref(c), C.byref(u)))
        return a.value, c.value, u.value

    def set_state(self, alpha, consumed, update_index):
        _chk(lib().vo_learner_set_state(self.h, alpha, consumed, update_index))


def adam_step(params, grads, m, v, step: int, lr: float) -> int:
    s = c_int64(step)
    for a in (params, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = np.ascontiguousarray(grads, np.float64)
    _chk(lib().vo_adam_step(params.size, _p(params, c_double), _p(g, c_double), _p(m, c_double),
                            _p(v, c_double), C.byref(s), lr))
    return s.value


def cosine_lr(base: float, total: int, consumed: int) -> float:
    return lib().vo_cosine_lr(base, total, consumed)


def estimate_time(tau, max_steps: int, steps: int) -> float:
    t = np.ascontiguousarray(tau, np.float64)
    out = c_double()
    _chk(lib().vo_estimate_time(_p(t, c_double), t.size, max_steps, steps, C.byref(out)))
    return out.value


def optimal_preempt_steps(tau, learn_time: float, max_steps: int) -> int:
    t = np.ascontiguousarray(tau, np.float64)
    out = c_int64()
    _chk(lib().vo_optimal_preempt_steps(_p(t, c_double), t.size, learn_time, max_steps, C.byref(out)))
    return out.value


def optimal_preempt_steps_sorted(tau, learn_time: float, max_steps: int) -> int:
    t = np.ascontiguousarray(tau, np.float64)
    out = c_int64()
    _chk(lib().vo_optimal_preempt_steps_sorted(_p(t, c_double), t.size, learn_time, max_steps,
                                               C.byref(out)))
    return out.value


def merged_time(tau, steps: int) -> float:
    t = np.ascontiguousarray(tau, np.float64)
    return lib().vo_merged_time(_p(t, c_double), t.size, steps)
