"""Host-side mirror of the reference's hot-path API over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj:
RolloutBuffer / close_rollout / backfill_stale (rollout.hpp:87-151),
split_minibatches / split_in_order / pack / unpack (packseq.hpp:35-44),
compute_gae / ppo_loss / Learner (learner.hpp:53-138), act / adam_step /
CosineSchedule (nn.hpp:67-118), estimate_time / optimal_preempt_steps
(distributed.hpp:29-32).  Every call goes through libver_b200.so; there is
no Python or CPU compute path.
"""
from __future__ import annotations

import ctypes as C
import sys as _sys
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib as L
from .hostview import HostView, SEQ_FIELDS

VER_OK, VER_ERR_PROTOCOL, VER_ERR_CONFIG, VER_ERR_NONFINITE, VER_ERR_CUDA, VER_ERR_NCCL = range(6)


class ProtocolError(RuntimeError):
    """ver::ProtocolError (types.hpp:41-44)."""


class ConfigError(RuntimeError):
    """ver::ConfigError (types.hpp:46-49)."""


class CudaError(RuntimeError):
    pass


def _check(status: int):
    if status == VER_OK:
        return
    msg = _lib().ver_last_error().decode(errors="replace")
    if status in (VER_ERR_PROTOCOL, VER_ERR_NONFINITE):
        raise ProtocolError(msg)
    if status == VER_ERR_CONFIG:
        raise ConfigError(msg)
    raise CudaError(f"[{status}] {msg}")


def _lib():
    return L.load()


def _ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ------------------------------------------------------------------ context
class Context:
    """One device + stream (+ optional NCCL communicator)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _check(_lib().ver_ctx_create(device, C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            _lib().ver_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(_lib().ver_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        s = C.c_uint64()
        _check(_lib().ver_ctx_stream(self.h, C.byref(s)))
        return s.value

    def launch_count(self, reset: bool = False) -> int:
        n = C.c_int64()
        _check(_lib().ver_ctx_launch_count(self.h, C.byref(n), int(reset)))
        return n.value

    def set_precision(self, mode: int):
        """0 = 3xTF32 tensor-core GEMMs (fp32-grade, default), 1 = 1xTF32 (fast)."""
        _check(_lib().ver_ctx_set_precision(self.h, mode))

    def set_tensor_cores(self, enable: bool):
        """True (default): tcgen05 GEMMs; False: fp32 SIMT GEMMs."""
        _check(_lib().ver_ctx_set_tensor_cores(self.h, int(enable)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib().ver_nccl_unique_id(buf))
        return buf.raw

    def init_nccl(self, uid: bytes, nranks: int, rank: int):
        _check(_lib().ver_ctx_init_nccl(self.h, uid, nranks, rank))

    def allreduce_sum_i64(self, values) -> np.ndarray:
        a = np.ascontiguousarray(values, dtype=np.int64).copy()
        _check(_lib().ver_allreduce_sum_i64(self.h, _ptr(a, C.c_int64), a.size))
        return a

    def allreduce_mean_f64(self, values) -> np.ndarray:
        a = np.ascontiguousarray(values, dtype=np.float64).copy()
        _check(_lib().ver_allreduce_mean_f64(self.h, _ptr(a, C.c_double), a.size))
        return a

    def allgather_f64(self, values, nranks: int) -> np.ndarray:
        a = np.ascontiguousarray(values, dtype=np.float64)
        out = np.zeros(a.size * nranks, np.float64)
        _check(_lib().ver_allgather_f64(self.h, _ptr(a, C.c_double), a.size, _ptr(out, C.c_double)))
        return out


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# --------------------------------------------------------------------- view
def _viewhost(hv: HostView, copy: bool = True) -> tuple[L.ViewHost, list]:
    """Build a ViewHost struct pointing into hv's arrays (float32 copies if `copy`)."""
    h = hv.astype(np.float32) if copy else hv
    keep = [h]
    vh = L.ViewHost()
    vh.T, vh.N, vh.action_kind = h.T, h.N, h.action_kind
    vh.obs_dim, vh.act_dim, vh.hidden_dim = h.obs_dim, h.act_dim, h.hidden_dim
    vh.size, vh.num_seqs, vh.h0_rows = h.size, h.num_seqs, h.h0.shape[0]
    vh.deficit, vh.stale_steps, vh.replayed_steps = h.deficit, h.stale_steps, h.replayed_steps
    vh.snapshot_version, vh.collect_wall_time = h.snapshot_version, h.collect_wall_time
    for name, ct in (("obs", C.c_float), ("act_cont", C.c_float), ("act_disc", C.c_int32),
                     ("log_prob", C.c_float), ("value", C.c_float), ("reward", C.c_float),
                     ("latency", C.c_float), ("advantage", C.c_float), ("returns", C.c_float),
                     ("done", C.c_uint8), ("stale", C.c_uint8), ("replayed", C.c_uint8),
                     ("env_index", C.c_int32), ("seq_of_slot", C.c_int32),
                     ("step_in_episode", C.c_int32), ("episode_index", C.c_int64),
                     ("version", C.c_uint64), ("h0", C.c_float), ("per_env_counts", C.c_int32),
                     ("env_bootstrap", C.c_float), ("env_bootstrap_valid", C.c_uint8)):
        a = getattr(h, name)
        setattr(vh, name, _ptr(a, ct) if a.size else None)
    vh.seqs = h.seqs.ctypes.data_as(C.POINTER(L.SeqDesc)) if h.seqs.size else None
    if h.action_kind == 0:
        vh.act_cont = None
    return vh, keep


class RolloutView:
    """Device-resident RolloutView handle (rollout.hpp:33-78)."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.h = handle
        self.ctx = ctx

    @staticmethod
    def from_host(hv: HostView, ctx: Context | None = None) -> "RolloutView":
        ctx = ctx or default_context()
        vh, keep = _viewhost(hv)
        out = C.c_void_p()
        _check(_lib().ver_view_upload(ctx.h, C.byref(vh), C.byref(out)))
        del keep
        return RolloutView(out, ctx)

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_view_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def info(self) -> L.ViewHost:
        vh = L.ViewHost()
        _check(_lib().ver_view_info(self.h, C.byref(vh)))
        return vh

    def size(self) -> int:
        return self.info().size

    def fresh_steps(self) -> int:
        i = self.info()
        return i.size - i.replayed_steps

    @property
    def deficit(self) -> int:
        return self.info().deficit

    @property
    def stale_steps(self) -> int:
        return self.info().stale_steps

    def to_host(self) -> HostView:
        i = self.info()
        hv = HostView.empty(i.T, i.N, i.action_kind, i.obs_dim, i.act_dim, i.hidden_dim, i.size,
                            i.num_seqs, i.h0_rows, fdtype=np.float32)
        hv.deficit, hv.stale_steps, hv.replayed_steps = i.deficit, i.stale_steps, i.replayed_steps
        hv.snapshot_version, hv.collect_wall_time = i.snapshot_version, i.collect_wall_time
        vh, _ = _viewhost(hv, copy=False)
        _check(_lib().ver_view_download(self.h, C.byref(vh)))
        return hv

    _FIELD_TYPES = {"obs": (np.float32, C.c_float, "S*D"), "log_prob": (np.float32, C.c_float, "S"),
                    "value": (np.float32, C.c_float, "S"), "reward": (np.float32, C.c_float, "S"),
                    "advantage": (np.float32, C.c_float, "S"), "returns": (np.float32, C.c_float, "S"),
                    "done": (np.uint8, C.c_uint8, "S"), "replayed": (np.uint8, C.c_uint8, "S"),
                    "env_index": (np.int32, C.c_int32, "S"), "act_disc": (np.int32, C.c_int32, "S"),
                    "per_env_counts": (np.int32, C.c_int32, "N"), "env_bootstrap": (np.float32, C.c_float, "N"),
                    "env_bootstrap_valid": (np.uint8, C.c_uint8, "N")}

    def fields(self, *names) -> dict:
        """Download only the named slot / env arrays (ver_view_download skips NULL fields)."""
        i = self.info()
        vh = L.ViewHost()
        vh.T, vh.N, vh.action_kind, vh.obs_dim, vh.act_dim, vh.hidden_dim = (i.T, i.N, i.action_kind, i.obs_dim,
                                                                             i.act_dim, i.hidden_dim)
        vh.size, vh.num_seqs, vh.h0_rows = i.size, i.num_seqs, i.h0_rows
        out = {}
        for n in names:
            dt, ct, shape = self._FIELD_TYPES[n]
            cnt = {"S": i.size, "N": i.N, "S*D": i.size * i.obs_dim}[shape]
            out[n] = np.empty(cnt, dt)
            setattr(vh, n, _ptr(out[n], ct))
        _check(_lib().ver_view_download(self.h, C.byref(vh)))
        return out

    def dump_jsonl(self, path):
        """dump_view (rollout.cpp:293-344): the reference's JSONL trace."""
        _check(_lib().ver_view_dump_jsonl(self.h, str(path).encode()))

    @staticmethod
    def load_jsonl(path, ctx: Context | None = None) -> "RolloutView":
        """load_view (rollout.cpp:346-432)."""
        ctx = ctx or default_context()
        out = C.c_void_p()
        _check(_lib().ver_view_load_jsonl(ctx.h, str(path).encode(), C.byref(out)))
        return RolloutView(out, ctx)

    def clone(self) -> "RolloutView":
        out = C.c_void_p()
        _check(_lib().ver_view_clone(self.h, C.byref(out)))
        return RolloutView(out, self.ctx)

    def restale(self, learner_version: int):
        _check(_lib().ver_view_restale(self.h, learner_version))


# ------------------------------------------------------------- rollout store
FIXED, VARIABLE = 0, 1
ACCEPTED, ROLLOUT_FULL = 0, 1


@dataclass
class StepRecords:
    """A batch of EnvStepRecords (types.hpp:54-67) in arrival order (SoA)."""
    env_index: np.ndarray
    obs: np.ndarray
    log_prob: np.ndarray
    value: np.ndarray
    reward: np.ndarray
    done: np.ndarray
    act_disc: np.ndarray | None = None
    act_cont: np.ndarray | None = None
    episode_index: np.ndarray | None = None
    step_in_episode: np.ndarray | None = None
    latency: np.ndarray | None = None
    h_before: np.ndarray | None = None
    h_before_valid: np.ndarray | None = None
    snapshot_version: np.ndarray | None = None

    def __len__(self):
        return int(np.asarray(self.env_index).shape[0])


class RolloutBuffer:
    """rollout.hpp:87-142 over the device store."""

    def __init__(self, T: int, N: int, mode: int = VARIABLE, action_kind: int = 0, obs_dim: int = 1,
                 act_dim: int = 0, hidden_dim: int = 0, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.cfg = L.RolloutConfig(T, N, mode, action_kind, obs_dim, act_dim, hidden_dim)
        self.h = C.c_void_p()
        _check(_lib().ver_rollout_create(self.ctx.h, C.byref(self.cfg), C.byref(self.h)))

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_rollout_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def begin_rollout(self, snapshot_version: int):
        _check(_lib().ver_rollout_begin(self.h, snapshot_version))

    def append_steps(self, recs: StepRecords) -> np.ndarray:
        n = len(recs)
        keep = []

        def arr(x, dt, shape=None):
            if x is None:
                return None
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a

        b = L.StepBatch()
        b.n = n
        b.env_index = _ptr(arr(recs.env_index, np.int32), C.c_int32)
        b.episode_index = _ptr(arr(recs.episode_index, np.int64), C.c_int64)
        b.step_in_episode = _ptr(arr(recs.step_in_episode, np.int32), C.c_int32)
        b.obs = _ptr(arr(recs.obs, np.float32), C.c_float)
        b.act_disc = _ptr(arr(recs.act_disc, np.int32), C.c_int32)
        b.act_cont = _ptr(arr(recs.act_cont, np.float32), C.c_float)
        b.log_prob = _ptr(arr(recs.log_prob, np.float32), C.c_float)
        b.value = _ptr(arr(recs.value, np.float32), C.c_float)
        b.reward = _ptr(arr(recs.reward, np.float32), C.c_float)
        b.latency = _ptr(arr(recs.latency, np.float32), C.c_float)
        b.done = _ptr(arr(recs.done, np.uint8), C.c_uint8)
        b.h_before = _ptr(arr(recs.h_before, np.float32), C.c_float)
        b.h_before_valid = _ptr(arr(recs.h_before_valid, np.uint8), C.c_uint8)
        b.snapshot_version = _ptr(arr(recs.snapshot_version, np.uint64), C.c_uint64)
        out = np.zeros(n, np.int32)
        _check(_lib().ver_rollout_append(self.h, C.byref(b), _ptr(out, C.c_int32)))
        return out

    def append_step(self, env: int, episode: int, t: int, obs, action, log_prob: float, value: float,
                    reward: float, done: bool, latency: float = 0.0, h_before=None,
                    snapshot_version: int = 0) -> int:
        cont = self.cfg.action_kind == 1
        recs = StepRecords(
            env_index=np.array([env]), obs=np.asarray(obs, np.float32).reshape(1, -1),
            log_prob=np.array([log_prob]), value=np.array([value]), reward=np.array([reward]),
            done=np.array([1 if done else 0]),
            act_disc=None if cont else np.array([int(action)]),
            act_cont=np.asarray(action, np.float32).reshape(1, -1) if cont else None,
            episode_index=np.array([episode]), step_in_episode=np.array([t]),
            latency=np.array([latency]),
            h_before=None if h_before is None else np.asarray(h_before, np.float32).reshape(1, -1),
            snapshot_version=np.array([snapshot_version], np.uint64))
        return int(self.append_steps(recs)[0])

    def force_close(self):
        _check(_lib().ver_rollout_force_close(self.h))

    def set_bootstrap(self, env: int, value: float):
        _check(_lib().ver_rollout_set_bootstrap(self.h, env, value))

    def set_bootstraps(self, envs, values):
        """set_bootstrap for many envs in one call."""
        e = np.ascontiguousarray(envs, np.int32)
        v = np.ascontiguousarray(values, np.float32)
        _check(_lib().ver_rollout_set_bootstraps(self.h, e.size, _ptr(e, C.c_int32), _ptr(v, C.c_float)))

    def _state(self):
        o, c, k = C.c_int(), C.c_int(), C.c_int()
        _check(_lib().ver_rollout_state(self.h, C.byref(o), C.byref(c), C.byref(k)))
        return o.value, c.value, k.value

    def open(self) -> bool:
        return bool(self._state()[0])

    def committed(self) -> int:
        return self._state()[1]

    def carryover_count(self) -> int:
        return self._state()[2]

    def capacity(self) -> int:
        return self.cfg.T * self.cfg.N

    def close_rollout(self) -> RolloutView:
        out = C.c_void_p()
        _check(_lib().ver_rollout_close(self.h, C.byref(out)))
        return RolloutView(out, self.ctx)


def view_synth(lengths, obs_dim: int = 2, hidden_dim: int = 4, seed: int = 1, p_done: float = 1.0 / 32,
               ctx: Context | None = None) -> RolloutView:
    """Device-generated ragged closed view (C5 stress workload)."""
    ctx = ctx or default_context()
    L_ = np.ascontiguousarray(lengths, dtype=np.int32)
    out = C.c_void_p()
    _check(_lib().ver_view_synth(ctx.h, _ptr(L_, C.c_int32), L_.size, obs_dim, hidden_dim, seed, p_done,
                                 C.byref(out)))
    return RolloutView(out, ctx)


def bench_gae_gather(view: RolloutView, B: int = 2, seed: int = 1, reps: int = 5, gamma: float = 0.99,
                     lam: float = 0.95, kernels: bool = False) -> tuple:
    """(GAE ms, gather ms for all B minibatches), CUDA-event timed around the
    calls; with kernels=True also (GAE scan kernel ms, gather kernels ms), timed
    around the launches alone."""
    ms = (C.c_float * 4)()
    _check(_lib().ver_bench_gae_gather(view.h, gamma, lam, B, seed, reps, ms))
    if kernels:
        return float(ms[0]), float(ms[1]), float(ms[2]), float(ms[3])
    return float(ms[0]), float(ms[1])


def backfill_stale(view: RolloutView, prev: RolloutView, deficit: int):
    _check(_lib().ver_backfill_stale(view.h, prev.h, deficit))


def compute_gae(view: RolloutView, gamma: float, lam: float):
    _check(_lib().ver_compute_gae(view.h, gamma, lam))


# ------------------------------------------------------------------ sampler
def _seqs_from(arr: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(arr, dtype=np.int32).reshape(-1, 8))


class SequenceGroup:
    """packseq.hpp:12-15.  Either a slice of a device deal or explicit host pieces."""

    def __init__(self, seqs: np.ndarray | None = None, total_steps: int | None = None,
                 _groups=None, _b: int = -1):
        self._groups = _groups
        self._b = _b
        if seqs is not None:
            self._seqs = _seqs_from(seqs)
            self.total_steps = int(self._seqs[:, 2].sum()) if total_steps is None else total_steps
        else:
            n, tot = C.c_int(), C.c_int()
            _check(_lib().ver_groups_get(_groups.h, _b, C.byref(n), C.byref(tot), None))
            self._seqs = None
            self._n = n.value
            self.total_steps = tot.value

    @property
    def seqs(self) -> np.ndarray:
        if self._seqs is None:
            a = np.zeros((self._n, 8), np.int32)
            if self._n:
                _check(_lib().ver_groups_get(self._groups.h, self._b, None, None,
                                             a.ctypes.data_as(C.POINTER(L.SeqDesc))))
            self._seqs = a
        return self._seqs

    def __len__(self):
        return self._n if self._seqs is None else self._seqs.shape[0]


class _Groups:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_groups_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass


def _groups_list(h) -> list[SequenceGroup]:
    g = _Groups(h)
    B = C.c_int()
    _check(_lib().ver_groups_count(h, C.byref(B)))
    return [SequenceGroup(_groups=g, _b=b) for b in range(B.value)]


def split_minibatches(view: RolloutView, B: int, seed: int) -> list[SequenceGroup]:
    out = C.c_void_p()
    _check(_lib().ver_split_minibatches(view.h, B, seed, C.byref(out)))
    return _groups_list(out)


def split_in_order(view: RolloutView, B: int, order: Sequence[int]) -> list[SequenceGroup]:
    o = np.ascontiguousarray(order, dtype=np.int32)
    out = C.c_void_p()
    _check(_lib().ver_split_in_order(view.h, B, _ptr(o, C.c_int32), o.size, C.byref(out)))
    return _groups_list(out)


class PackedBatch:
    """packseq.hpp:20-29 (device) + the gathered time-major learner fields."""

    def __init__(self, h, view: RolloutView):
        self.h = h
        self.view = view
        k, L_, S = C.c_int(), C.c_int(), C.c_int()
        _check(_lib().ver_packed_info(h, C.byref(k), C.byref(L_), C.byref(S)))
        self.num_seqs, self._max_len, self.total_steps = k.value, L_.value, S.value
        self._cache = None

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_packed_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def max_len(self) -> int:
        return self._max_len

    def _load(self):
        if self._cache is None:
            seqs = np.zeros((self.num_seqs, 8), np.int32)
            s2g = np.zeros(self.num_seqs, np.int32)
            bs = np.zeros(self._max_len, np.int32)
            offs = np.zeros(self._max_len, np.int32)
            slots = np.zeros(self.total_steps, np.int32)
            _check(_lib().ver_packed_get(self.h, seqs.ctypes.data_as(C.POINTER(L.SeqDesc)),
                                         _ptr(s2g, C.c_int32), _ptr(bs, C.c_int32),
                                         _ptr(offs, C.c_int32), _ptr(slots, C.c_int32)))
            self._cache = (seqs, s2g, bs, offs, slots)
        return self._cache

    @property
    def seqs(self):
        return self._load()[0]

    @property
    def sorted_to_group(self):
        return self._load()[1]

    @property
    def batch_sizes(self):
        return self._load()[2]

    @property
    def offsets(self):
        return self._load()[3]

    @property
    def slots(self):
        return self._load()[4]

    def gathered(self, obs_dim: int, action_kind: int = 0, act_dim: int = 0) -> dict:
        S = self.total_steps
        obs = np.zeros((S, obs_dim), np.float32)
        act = np.zeros(S, np.int32) if action_kind == 0 else None
        actc = np.zeros((S, act_dim), np.float32) if action_kind == 1 else None
        lp, adv, ret = (np.zeros(S, np.float32) for _ in range(3))
        _check(_lib().ver_packed_get_gathered(self.h, _ptr(obs, C.c_float), _ptr(act, C.c_int32),
                                              _ptr(actc, C.c_float), _ptr(lp, C.c_float),
                                              _ptr(adv, C.c_float), _ptr(ret, C.c_float)))
        return dict(obs=obs, act_disc=act, act_cont=actc, old_logp=lp, adv=adv, ret=ret)


def pack(view: RolloutView, group: SequenceGroup) -> PackedBatch:
    out = C.c_void_p()
    if group._groups is not None:
        _check(_lib().ver_pack(view.h, group._groups.h, group._b, C.byref(out)))
    else:
        s = group._seqs
        _check(_lib().ver_pack_seqs(view.h, s.ctypes.data_as(C.POINTER(L.SeqDesc)) if s.size else None,
                                    s.shape[0], C.byref(out)))
    return PackedBatch(out, view)


def unpack(batch: PackedBatch) -> list[list[int]]:
    """packseq.cpp:90-101 — test oracle over the downloaded layout."""
    seqs, s2g, bs, offs, slots = batch._load()
    out: list[list[int]] = [[] for _ in range(batch.num_seqs)]
    for j in range(batch.num_seqs):
        gi = int(s2g[j])
        out[gi] = [int(slots[offs[t] + j]) for t in range(int(seqs[j, 2]))]
    return out


# ------------------------------------------------------------------- model
@dataclass
class ModelConfig:
    obs_dim: int
    encoder_dim: int = 64
    hidden_dim: int = 64
    action_kind: int = 0
    num_actions: int = 0
    act_dim: int = 0

    def c(self) -> L.ModelConfig:
        return L.ModelConfig(self.obs_dim, self.encoder_dim, self.hidden_dim, self.action_kind,
                             self.num_actions, self.act_dim)


def param_count(cfg: ModelConfig) -> int:
    n = C.c_int64()
    _check(_lib().ver_param_count(C.byref(cfg.c()), C.byref(n), None))
    return n.value


def param_tensors(cfg: ModelConfig) -> list[tuple[str, int, int, int]]:
    """[(name, rows, cols, offset)] in PolicyParams::tensors() order."""
    nt = C.c_int()
    _check(_lib().ver_param_count(C.byref(cfg.c()), None, C.byref(nt)))
    out = []
    for i in range(nt.value):
        name = C.create_string_buffer(16)
        r, c_, o = C.c_int(), C.c_int(), C.c_int64()
        _check(_lib().ver_param_tensor(C.byref(cfg.c()), i, name, C.byref(r), C.byref(c_), C.byref(o)))
        out.append((name.value.decode(), r.value, c_.value, o.value))
    return out


def params_init(cfg: ModelConfig, seed: int) -> np.ndarray:
    """PolicyParams::init (nn.cpp:16-81) — flat float64 in tensors() order."""
    out = np.zeros(param_count(cfg), np.float64)
    _check(_lib().ver_params_init(C.byref(cfg.c()), seed, _ptr(out, C.c_double)))
    return out


@dataclass
class PPOConfig:
    gamma: float = 0.99
    gae_lambda: float = 0.95
    clip: float = 0.2
    epochs: int = 3
    minibatches: int = 2
    value_loss_coef: float = 0.5
    is_cap: float = 1.0

    def c(self) -> L.PPOConfig:
        return L.PPOConfig(self.gamma, self.gae_lambda, self.clip, self.epochs, self.minibatches,
                           self.value_loss_coef, self.is_cap)


@dataclass
class EntropyController:
    """learner.hpp:29-40."""
    alpha: float = 1e-3
    target: float = 0.0
    lower: float = 1e-4
    upper: float = 1.0
    lr: float = 2.5e-4

    def update(self, mean_entropy: float):
        self.alpha += self.lr * (self.target - mean_entropy)
        self.alpha = min(max(self.alpha, self.lower), self.upper)

    def c(self) -> L.EntropyController:
        return L.EntropyController(self.alpha, self.target, self.lower, self.upper, self.lr)


def entropy_loss_value(mean_entropy: float, c: EntropyController) -> float:
    return c.alpha * (c.target - mean_entropy) - c.alpha * mean_entropy


@dataclass
class CosineSchedule:
    base_lr: float = 2.5e-4
    total_steps: int = 1

    def lr_at(self, consumed: int) -> float:
        return _lib().ver_cosine_lr(self.base_lr, self.total_steps, consumed)


@dataclass
class PPOLossResult:
    loss: float
    policy_loss: float
    value_loss: float
    mean_entropy: float
    ratio_sum: float
    clip_count: float
    w_sum: float
    w_max: float
    steps: int
    is_weights: np.ndarray
    grads: np.ndarray | None


def ppo_loss(cfg: ModelConfig, params: np.ndarray, view: RolloutView, batch: PackedBatch,
             ppo: PPOConfig, alpha: float, h0_sorted: np.ndarray, want_grads: bool = True,
             frozen_is_weights: np.ndarray | None = None,
             ctx: Context | None = None) -> PPOLossResult:
    ctx = ctx or view.ctx
    p = _f32(params)
    h0 = _f32(h0_sorted)
    fw = None if frozen_is_weights is None else _f32(frozen_is_weights).reshape(-1)
    res = L.LossResult()
    grads = np.zeros(p.size, np.float32) if want_grads else None
    isw = np.zeros(batch.total_steps, np.float32)
    _check(_lib().ver_ppo_loss(ctx.h, C.byref(cfg.c()), _ptr(p, C.c_float), view.h, batch.h,
                               C.byref(ppo.c()), alpha, _ptr(h0, C.c_float), int(want_grads),
                               _ptr(fw, C.c_float), C.byref(res), _ptr(grads, C.c_float),
                               _ptr(isw, C.c_float)))
    return PPOLossResult(res.loss, res.policy_loss, res.value_loss, res.mean_entropy, res.ratio_sum,
                         res.clip_count, res.w_sum, res.w_max, res.steps, isw, grads)


def forward_packed(cfg: ModelConfig, params: np.ndarray, obs: np.ndarray, act_disc, act_cont,
                   batch_sizes, offsets, h0: np.ndarray, ctx: Context | None = None):
    """nn.cpp:219-280 -> (log_prob, entropy, value) per packed row."""
    ctx = ctx or default_context()
    obs = _f32(obs).reshape(-1, cfg.obs_dim)
    S = obs.shape[0]
    bs = np.ascontiguousarray(batch_sizes, np.int32)
    of = np.ascontiguousarray(offsets, np.int32)
    h0 = _f32(h0).reshape(-1, cfg.hidden_dim)
    ad = None if act_disc is None else np.ascontiguousarray(act_disc, np.int32)
    ac = None if act_cont is None else _f32(act_cont)
    lp, en, va = (np.zeros(S, np.float32) for _ in range(3))
    p = _f32(params)
    _check(_lib().ver_forward_packed(ctx.h, C.byref(cfg.c()), _ptr(p, C.c_float), S, _ptr(obs, C.c_float),
                                     _ptr(ad, C.c_int32), _ptr(ac, C.c_float), bs.size, _ptr(bs, C.c_int32),
                                     _ptr(of, C.c_int32), _ptr(h0, C.c_float), _ptr(lp, C.c_float),
                                     _ptr(en, C.c_float), _ptr(va, C.c_float)))
    return lp, en, va


def act(cfg: ModelConfig, params: np.ndarray, obs: np.ndarray, h: np.ndarray,
        ctx: Context | None = None):
    """nn.cpp:118-126 -> (dist, value, h_new)."""
    ctx = ctx or default_context()
    obs = _f32(obs).reshape(-1, cfg.obs_dim)
    h = _f32(h).reshape(-1, cfg.hidden_dim)
    n = obs.shape[0]
    A = cfg.num_actions if cfg.action_kind == 0 else cfg.act_dim
    dist = np.zeros((n, A), np.float32)
    val = np.zeros(n, np.float32)
    hn = np.zeros((n, cfg.hidden_dim), np.float32)
    p = _f32(params)
    _check(_lib().ver_act(ctx.h, C.byref(cfg.c()), _ptr(p, C.c_float), n, _ptr(obs, C.c_float),
                          _ptr(h, C.c_float), _ptr(dist, C.c_float), _ptr(val, C.c_float),
                          _ptr(hn, C.c_float)))
    return dist, val, hn


def adam_step(params: np.ndarray, grads: np.ndarray, m: np.ndarray, v: np.ndarray, step: int,
              lr: float, ctx: Context | None = None) -> int:
    """nn.cpp:291-306 on float32 arrays in place; returns the new step."""
    ctx = ctx or default_context()
    for a in (params, m, v):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    g = _f32(grads)
    s = C.c_int64(step)
    _check(_lib().ver_adam_step(ctx.h, params.size, _ptr(params, C.c_float), _ptr(g, C.c_float),
                                _ptr(m, C.c_float), _ptr(v, C.c_float), C.byref(s), lr))
    return s.value


@dataclass
class TrainStats:
    update_index: int
    steps: int
    fresh_steps: int
    stale_steps: int
    loss: float
    policy_loss: float
    value_loss: float
    entropy: float
    entropy_loss: float
    mean_ratio: float
    clip_fraction: float
    mean_is_weight: float
    max_is_weight: float
    alpha: float
    lr: float


class DeviceBuffer:
    """A library-owned fp32 device array handed to a learner hook: ``ptr``
    (device address), ``count`` floats, the ctx ``stream`` (cudaStream_t as int).
    ``__cuda_array_interface__`` lets torch / cupy wrap it without a copy."""

    def __init__(self, ptr: int, count: int, stream: int, device: int):
        self.ptr, self.count, self.stream, self.device = int(ptr or 0), int(count), int(stream), device

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.count,), "typestr": "<f4", "data": (self.ptr, False), "version": 3,
                "stream": self.stream or None}

    def torch(self):
        import torch
        return torch.as_tensor(self, device=f"cuda:{self.device}")


def param_device_index(cfg: ModelConfig) -> np.ndarray:
    """index[k] = device-layout position of the tensors()-order parameter k."""
    out = np.zeros(param_count(cfg), np.int64)
    _check(_lib().ver_param_device_index(C.byref(cfg.c()), _ptr(out, C.c_int64)))
    return out


PHASES = ("gae", "sampler", "replay", "forward", "loss", "backward", "allreduce", "adam", "rec_fwd", "rec_bwd",
          "gemm_fwd", "gemm_bwd")


class Learner:
    """learner.hpp:102-138 — owns params, Adam state and alpha on the device."""

    def __init__(self, cfg: ModelConfig, params: np.ndarray, ppo: PPOConfig = PPOConfig(),
                 entropy: EntropyController = EntropyController(),
                 schedule: CosineSchedule = CosineSchedule(), run_seed: int = 0,
                 ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.cfg = cfg
        self.ppo = ppo
        self.entropy_cfg = entropy
        self.h = C.c_void_p()
        p = _f32(params)
        _check(_lib().ver_learner_create(self.ctx.h, C.byref(cfg.c()), _ptr(p, C.c_float),
                                         C.byref(ppo.c()), C.byref(entropy.c()), schedule.base_lr,
                                         schedule.total_steps, run_seed, C.byref(self.h)))
        self.P = p.size

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_learner_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def enable_allreduce(self, on: bool = True):
        _check(_lib().ver_learner_enable_allreduce(self.h, int(on)))

    def set_hooks(self, grad_hook=None, entropy_hook=None):
        """Learner::grad_hook / entropy_hook (learner.hpp:119-122).

        Each hook is called once per minibatch between backward and Adam with a
        :class:`DeviceBuffer` (the P gradients in device layout, or the one-float
        minibatch mean entropy) and must average it in place before returning
        (the buffer exposes ``__cuda_array_interface__`` and the ctx stream)."""
        def wrap_g(fn):
            if fn is None:
                return L.GradHook()

            def cb(_user, ptr, n, stream):
                try:
                    fn(DeviceBuffer(ptr, n, stream, self.ctx.device))
                    return 0
                except Exception as e:  # reported as VER_ERR_CONFIG by the update
                    self._hook_error = e
                    return 1
            return L.GradHook(cb)

        def wrap_h(fn):
            if fn is None:
                return L.EntropyHook()

            def cb(_user, ptr, stream):
                try:
                    fn(DeviceBuffer(ptr, 1, stream, self.ctx.device))
                    return 0
                except Exception as e:
                    self._hook_error = e
                    return 1
            return L.EntropyHook(cb)

        self._hooks = (wrap_g(grad_hook), wrap_h(entropy_hook))  # keep the thunks alive
        _check(_lib().ver_learner_set_grad_hook(self.h, self._hooks[0], None))
        _check(_lib().ver_learner_set_entropy_hook(self.h, self._hooks[1], None))

    def update(self, view: RolloutView, read_stats: bool = True) -> TrainStats | None:
        if not read_stats:
            _check(_lib().ver_learner_update(self.h, view.h, None))
            return None
        s = L.TrainStats()
        _check(_lib().ver_learner_update(self.h, view.h, C.byref(s)))
        return TrainStats(*(getattr(s, f) for f, _ in L.TrainStats._fields_))

    def batch_h0(self, view: RolloutView, batch: PackedBatch) -> np.ndarray:
        out = np.zeros((batch.num_seqs, self.cfg.hidden_dim), np.float32)
        _check(_lib().ver_learner_batch_h0(self.h, view.h, batch.h, _ptr(out, C.c_float)))
        return out

    def params(self) -> np.ndarray:
        out = np.zeros(self.P, np.float32)
        _check(_lib().ver_learner_get_params(self.h, _ptr(out, C.c_float)))
        return out

    def set_params(self, p: np.ndarray):
        p = _f32(p)
        _check(_lib().ver_learner_set_params(self.h, _ptr(p, C.c_float)))

    def adam(self):
        m = np.zeros(self.P, np.float32)
        v = np.zeros(self.P, np.float32)
        s = C.c_int64()
        _check(_lib().ver_learner_get_adam(self.h, _ptr(m, C.c_float), _ptr(v, C.c_float), C.byref(s)))
        return m, v, s.value

    def set_adam(self, m, v, step: int):
        m, v = _f32(m), _f32(v)
        _check(_lib().ver_learner_set_adam(self.h, _ptr(m, C.c_float), _ptr(v, C.c_float), step))

    def _state(self):
        a, c, u = C.c_double(), C.c_int64(), C.c_int64()
        _check(_lib().ver_learner_get_state(self.h, C.byref(a), C.byref(c), C.byref(u)))
        return a.value, c.value, u.value

    @property
    def alpha(self) -> float:
        return self._state()[0]

    def consumed_steps(self) -> int:
        return self._state()[1]

    def update_index(self) -> int:
        return self._state()[2]

    def set_state(self, alpha=None, consumed=None, update_index=None):
        a, c, u = self._state()
        _check(_lib().ver_learner_set_state(self.h, a if alpha is None else alpha,
                                            c if consumed is None else consumed,
                                            u if update_index is None else update_index))

    def save_checkpoint(self, path):
        """save_checkpoint (bench.cpp:411-424): "ver-checkpoint" v1 JSON."""
        _check(_lib().ver_learner_save_checkpoint(self.h, str(path).encode()))

    def load_checkpoint(self, path):
        """load_checkpoint (bench.cpp:426-441) into this learner (same model)."""
        _check(_lib().ver_learner_load_checkpoint(self.h, str(path).encode()))

    def set_consumed_steps(self, n: int):
        self.set_state(consumed=n)

    def set_update_index(self, n: int):
        self.set_state(update_index=n)

    def last_timing(self) -> dict:
        ms = (C.c_float * 16)()
        n = C.c_int(16)
        _check(_lib().ver_learner_last_timing(self.h, ms, C.byref(n)))
        return {PHASES[i]: float(ms[i]) for i in range(min(n.value, len(PHASES)))}

    def last_flop(self) -> dict:
        """Algorithmic FLOPs (2MNK) of the tcgen05 GEMM launches of the last update per phase."""
        f = (C.c_double * 16)()
        n = C.c_int(16)
        _check(_lib().ver_learner_last_flop(self.h, f, C.byref(n)))
        return {PHASES[i]: float(f[i]) for i in range(min(n.value, len(PHASES)))}

    def last_timing_counts(self) -> dict:
        """Intervals behind each phase of last_timing (launches for rec_fwd / rec_bwd)."""
        cnt = (C.c_int * 16)()
        n = C.c_int(16)
        _check(_lib().ver_learner_last_timing_counts(self.h, cnt, C.byref(n)))
        return {PHASES[i]: int(cnt[i]) for i in range(min(n.value, len(PHASES)))}


@dataclass
class IterationResult:
    """IterationResult (distributed.hpp:138-147) of one ver_replica_learn."""
    iteration: int
    rank: int
    deficit: int
    stale_steps: int
    global_consumed_before: int
    global_fresh: int
    learn_time: float
    mean_learn_time: float
    next_threshold: int
    per_replica_threshold: int
    train: TrainStats


PREEMPT_NONE, PREEMPT_OPTIMAL = 0, 1


class Replica:
    """The learner section of ReplicaGroup::replica_main (distributed.cpp:208-264)
    for one process per GPU (csrc/replica.cu).

    ``comm=None`` uses NCCL on the learner's context (``Context.init_nccl``); or
    pass an object with ``nranks``, ``rank`` and host-side ``sum_i64(arr)``,
    ``mean_f64(arr)`` (in place) and ``allgather_f64(arr) -> array`` methods."""

    def __init__(self, learner: "Learner", T: int, N: int, preempt: int = PREEMPT_OPTIMAL,
                 per_replica_budget: bool = False, comm=None):
        self.learner = learner
        self.ctx = learner.ctx
        self.h = C.c_void_p()
        cfg = L.ReplicaConfig(T, N, preempt, int(per_replica_budget))
        cp = None
        if comm is not None:
            self._comm_obj = comm

            def sum_i64(_u, p, n):
                try:
                    a = np.ctypeslib.as_array(p, shape=(n,))
                    comm.sum_i64(a)
                    return 0
                except Exception:
                    return 1

            def mean_f64(_u, p, n):
                try:
                    a = np.ctypeslib.as_array(p, shape=(n,))
                    comm.mean_f64(a)
                    return 0
                except Exception:
                    return 1

            def allgather(_u, p, n, out):
                try:
                    a = np.ctypeslib.as_array(p, shape=(n,)).copy()
                    o = np.ctypeslib.as_array(out, shape=(n * comm.nranks,))
                    o[:] = comm.allgather_f64(a)
                    return 0
                except Exception:
                    return 1

            self._thunks = (L.SumI64(sum_i64), L.MeanF64(mean_f64), L.AllgatherF64(allgather))
            cp = L.ReplicaComm(None, *self._thunks, comm.nranks, comm.rank)
        _check(_lib().ver_replica_create(self.ctx.h, learner.h, C.byref(cfg), C.byref(cp) if cp else None,
                                         C.byref(self.h)))

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_replica_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def attach_preempt(self, counter: "PreemptCounter"):
        self._counter = counter
        _check(_lib().ver_replica_attach_preempt(self.h, counter.h))

    def learn(self, view: RolloutView, collect_wall_time: float = -1.0, last_iteration: bool = False
              ) -> IterationResult:
        r = L.IterationResult()
        _check(_lib().ver_replica_learn(self.h, view.h, collect_wall_time, int(last_iteration), C.byref(r)))
        tr = TrainStats(*(getattr(r.train, f) for f, _ in L.TrainStats._fields_))
        return IterationResult(r.iteration, r.rank, r.deficit, r.stale_steps, r.global_consumed_before,
                               r.global_fresh, r.learn_time, r.mean_learn_time, r.next_threshold,
                               r.per_replica_threshold, tr)

    def state(self) -> tuple[int, int, bool]:
        g, i, hp = C.c_int64(), C.c_int64(), C.c_int()
        _check(_lib().ver_replica_state(self.h, C.byref(g), C.byref(i), C.byref(hp)))
        return g.value, i.value, bool(hp.value)


def debug_gemm(A, B, transA=False, transB=False, engine=1, splitk=1, ctx: Context | None = None):
    """C = op(A) op(B) through the library GEMM (engine 0 SIMT, 1 tcgen05 3xTF32, 2 tcgen05 1xTF32)."""
    ctx = ctx or default_context()
    A = _f32(A)
    B = _f32(B)
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    C_ = np.zeros((M, N), np.float32)
    _check(_lib().ver_debug_gemm(ctx.h, engine, int(transA), int(transB), M, N, K, _ptr(A, C.c_float),
                                 A.shape[1], _ptr(B, C.c_float), B.shape[1], _ptr(C_, C.c_float), splitk))
    return C_


def debug_gemm_time(M, N, K, transA=False, transB=False, engine=1, splitk=1, reps=10,
                    ctx: Context | None = None) -> float:
    """Device ms per GEMM of this shape through the library GEMM (operands resident)."""
    ctx = ctx or default_context()
    ms = (C.c_float * 1)()
    _check(_lib().ver_debug_gemm_time(ctx.h, engine, int(transA), int(transB), M, N, K, splitk, reps, ms))
    return float(ms[0])


def debug_gemm_prof(on: bool, ctx: Context | None = None) -> list[int]:
    """tcgen05 GEMM wait-cycle counters (tc_gemm.cuh g_tc_prof); returns the sums so far."""
    ctx = ctx or default_context()
    out = (C.c_ulonglong * 16)()
    _check(_lib().ver_debug_gemm_prof(ctx.h, int(on), out))
    return [int(x) for x in out]


# ---------------------------------------------------------- distributed
def estimate_time(step_times, max_steps: int, steps: int, ctx: Context | None = None) -> float:
    ctx = ctx or default_context()
    t = np.ascontiguousarray(step_times, dtype=np.float64)
    out = C.c_double()
    _check(_lib().ver_estimate_time(ctx.h, _ptr(t, C.c_double), t.size, max_steps, steps, C.byref(out)))
    return out.value


def optimal_preempt_steps(step_times, learn_time: float, max_steps: int,
                          ctx: Context | None = None) -> int:
    ctx = ctx or default_context()
    t = np.ascontiguousarray(step_times, dtype=np.float64)
    out = C.c_int64()
    _check(_lib().ver_optimal_preempt_steps(ctx.h, _ptr(t, C.c_double), t.size, learn_time, max_steps,
                                            C.byref(out)))
    return out.value




def checkpoint_model_config(path) -> ModelConfig:
    """The model config stored in a "ver-checkpoint" file (nn.cpp:339-348)."""
    mc = L.ModelConfig()
    _check(_lib().ver_checkpoint_model_config(str(path).encode(), C.byref(mc)))
    return ModelConfig(obs_dim=mc.obs_dim, encoder_dim=mc.encoder_dim, hidden_dim=mc.hidden_dim,
                       action_kind=mc.action_kind, num_actions=mc.num_actions, act_dim=mc.act_dim)


# ------------------------------------------------------ preemption counter
class PreemptCounter:
    """PreemptCoordinator (distributed.hpp:95-128) across processes.

    IPC mode (default): one replica creates the device counter and exports its
    IPC handle (64 bytes); the others open it.  add_steps returns (total,
    fired_now); exactly one add per iteration fires.  NCCL mode (nccl=True, ctx
    with NCCL initialised, one counter per rank): adds accumulate locally and
    tick() -- a collective all ranks call once per collection tick -- sums them
    with ncclAllReduce, so all ranks fire on the same tick.  An InferenceEngine
    attached with attach_preempt() adds each batch's commits from its sampling
    kernel and force-closes its rollout once the group has fired."""

    def __init__(self, ctx: Context | None = None, handle: bytes | None = None, nccl: bool = False):
        self.ctx = ctx or default_context()
        self.h = C.c_void_p()
        self.nccl = nccl
        if nccl:
            _check(_lib().ver_preempt_create_nccl(self.ctx.h, C.byref(self.h)))
            self.owner = True
        elif handle is None:
            _check(_lib().ver_preempt_create(self.ctx.h, C.byref(self.h)))
            self.owner = True
        else:
            buf = (C.c_uint8 * 64).from_buffer_copy(bytes(handle))
            _check(_lib().ver_preempt_open(self.ctx.h, buf, C.byref(self.h)))
            self.owner = False

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_preempt_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        _check(_lib().ver_preempt_ipc_handle(self.h, buf))
        return bytes(buf)

    def start_iteration(self, threshold: int):
        _check(_lib().ver_preempt_start(self.h, threshold))

    def add_steps(self, n: int) -> tuple[int, bool]:
        t, f = C.c_int64(), C.c_int()
        _check(_lib().ver_preempt_add(self.h, n, C.byref(t), C.byref(f)))
        return t.value, bool(f.value)

    def state(self) -> tuple[int, bool]:
        t, f = C.c_int64(), C.c_int()
        _check(_lib().ver_preempt_state(self.h, C.byref(t), C.byref(f)))
        return t.value, bool(f.value)

    def tick(self) -> tuple[int, bool]:
        """NCCL mode: (global total, fired on this tick); collective over the ranks."""
        t, f = C.c_int64(), C.c_int()
        _check(_lib().ver_preempt_tick(self.h, C.byref(t), C.byref(f)))
        return t.value, bool(f.value)


# --------------------------------------------------------- inference engine
@dataclass
class InferenceRequest:
    """runtime.hpp:30-42."""
    env_index: int
    observation: np.ndarray
    reward: float = 0.0
    done: bool = False
    first: bool = False
    latency: float = 0.0
    obs_episode: int = 0
    obs_step: int = 0


@dataclass
class BatchResult:
    """InferenceEngine::BatchResult (runtime.hpp:98-106): dispatches = [(env, action)]."""
    dispatches: list
    new_commits: int = 0
    closed_now: bool = False
    preempt_fired: bool = False


class InferenceEngine:
    """InferenceEngine (runtime.hpp:96-160) on the device: batched act + on-device
    sampling with the reference's counter-RNG streams; every env's GRU state and
    the pending h_before stay in device memory; completed steps go into the
    engine's own rollout store (closed with close())."""

    def __init__(self, model: ModelConfig, T: int, N: int, params: np.ndarray, version: int = 0,
                 mode: int = VARIABLE, seed: int = 0, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.model = model
        self.N = N
        mc = model.c()
        rc = L.RolloutConfig(T, N, mode, model.action_kind, model.obs_dim,
                             model.act_dim if model.action_kind == 1 else 0, model.hidden_dim)
        self.cfg = L.EngineConfig(rc, mc, seed)
        self.h = C.c_void_p()
        p = _f32(params)
        _check(_lib().ver_engine_create(self.ctx.h, C.byref(self.cfg), _ptr(p, C.c_float), version,
                                        C.byref(self.h)))

    def __del__(self):
        if _sys.is_finalizing():
            return
        try:
            if self.h:
                _lib().ver_engine_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def set_snapshot(self, params, version: int):
        p = _f32(params)
        _check(_lib().ver_engine_set_snapshot(self.h, _ptr(p, C.c_float), version))

    def set_snapshot_from(self, learner: "Learner", version: int):
        """Device-to-device snapshot of a learner's current parameters."""
        _check(_lib().ver_engine_set_snapshot_learner(self.h, learner.h, version))

    def _result(self, r: L.BatchResult, env, act_d, act_c) -> BatchResult:
        n = r.n_dispatch
        if self.model.action_kind == 1:
            d = [(int(env[i]), act_c[i].copy()) for i in range(n)]
        else:
            d = [(int(env[i]), int(act_d[i])) for i in range(n)]
        return BatchResult(d, r.new_commits, bool(r.closed_now), bool(r.preempt_fired))

    def _bufs(self, n: int):
        A = max(1, self.model.act_dim if self.model.action_kind == 1 else 1)
        return (np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32),
                np.zeros((max(n, 1), A), np.float32))

    def begin_rollout(self) -> BatchResult:
        env, ad, ac = self._bufs(self.N)
        r = L.BatchResult()
        _check(_lib().ver_engine_begin_rollout(self.h, C.byref(r), _ptr(env, C.c_int32), _ptr(ad, C.c_int32),
                                               _ptr(ac, C.c_float)))
        return self._result(r, env, ad, ac)

    def process_batch(self, reqs: Sequence[InferenceRequest]) -> BatchResult:
        n = len(reqs)
        D = self.model.obs_dim
        envs = np.array([q.env_index for q in reqs], np.int32)
        obs = np.zeros((max(n, 1), D), np.float32)
        for i, q in enumerate(reqs):
            obs[i] = np.asarray(q.observation, np.float32).reshape(D)
        rw = np.array([q.reward for q in reqs], np.float32)
        dn = np.array([1 if q.done else 0 for q in reqs], np.uint8)
        fs = np.array([1 if q.first else 0 for q in reqs], np.uint8)
        lat = np.array([q.latency for q in reqs], np.float32)
        oe = np.array([q.obs_episode for q in reqs], np.int64)
        os_ = np.array([q.obs_step for q in reqs], np.int32)
        b = L.RequestBatch(n, _ptr(envs, C.c_int32), _ptr(obs, C.c_float), _ptr(rw, C.c_float),
                           _ptr(dn, C.c_uint8), _ptr(fs, C.c_uint8), _ptr(lat, C.c_float),
                           _ptr(oe, C.c_int64), _ptr(os_, C.c_int32))
        env, ad, ac = self._bufs(n)
        r = L.BatchResult()
        _check(_lib().ver_engine_process_batch(self.h, C.byref(b), C.byref(r), _ptr(env, C.c_int32),
                                               _ptr(ad, C.c_int32), _ptr(ac, C.c_float)))
        return self._result(r, env, ad, ac)

    def process_arrays(self, env, obs, reward=None, done=None, first=None, latency=None, obs_episode=None,
                       obs_step=None):
        """process_batch over SoA host arrays (no per-request Python objects):
        returns (BatchResult counts, dispatch env array, dispatch action array)."""
        n = int(np.asarray(env).size)
        keep = []

        def arr(x, dt):
            if x is None:
                return None
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a

        b = L.RequestBatch(n, _ptr(arr(env, np.int32), C.c_int32), _ptr(arr(obs, np.float32), C.c_float),
                           _ptr(arr(reward, np.float32), C.c_float), _ptr(arr(done, np.uint8), C.c_uint8),
                           _ptr(arr(first, np.uint8), C.c_uint8), _ptr(arr(latency, np.float32), C.c_float),
                           _ptr(arr(obs_episode, np.int64), C.c_int64), _ptr(arr(obs_step, np.int32), C.c_int32))
        de, ad, ac = self._bufs(n)
        r = L.BatchResult()
        _check(_lib().ver_engine_process_batch(self.h, C.byref(b), C.byref(r), _ptr(de, C.c_int32),
                                               _ptr(ad, C.c_int32), _ptr(ac, C.c_float)))
        k = r.n_dispatch
        return r, de[:k], (ac[:k] if self.model.action_kind == 1 else ad[:k])

    def force_close(self):
        _check(_lib().ver_engine_force_close(self.h))

    def attach_preempt(self, counter: "PreemptCounter | None"):
        """Joint preemption (runtime.cpp:592-599): each batch's commits go to
        `counter` from the sampling kernel; the first batch that sees the group
        fired force-closes this rollout.  None detaches."""
        self._preempt = counter  # keep the handle alive while attached
        _check(_lib().ver_engine_attach_preempt(self.h, counter.h if counter is not None else None))

    def finalize_bootstraps(self):
        _check(_lib().ver_engine_finalize_bootstraps(self.h))

    def close(self) -> RolloutView:
        out = C.c_void_p()
        _check(_lib().ver_engine_close(self.h, C.byref(out)))
        return RolloutView(out, self.ctx)

    def _state(self):
        v = [C.c_int() for _ in range(5)]
        _check(_lib().ver_engine_state(self.h, *[C.byref(x) for x in v]))
        return [x.value for x in v]

    def rollout_done(self) -> bool:
        return not self._state()[0]

    def committed(self) -> int:
        return self._state()[1]

    def capacity(self) -> int:
        return self._state()[2]

    def carryover_count(self) -> int:
        return self._state()[3]

    def active_envs(self) -> int:
        return self._state()[4]

    def hidden(self) -> np.ndarray:
        h = np.zeros((self.N, self.model.hidden_dim), np.float32)
        _check(_lib().ver_engine_hidden(self.h, _ptr(h, C.c_float)))
        return h


__all__ = [n for n in dir() if not n.startswith("_")] + ["SEQ_FIELDS"]
