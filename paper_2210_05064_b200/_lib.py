"""ctypes binding of the C-ABI in include/ver_gpu.h (libver_b200.so).

The library is loaded from the package's ``_lib/`` directory only; if it is
missing the import fails loudly — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libver_b200.so"

c_int, c_int32, c_int64, c_uint64, c_float, c_double = (
    C.c_int, C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double)
P = C.POINTER


class SeqDesc(C.Structure):
    _fields_ = [(n, c_int32) for n in ("seq_id", "env_index", "length", "start_offset", "h0_index",
                                        "stale", "parent_start_offset", "skip")]


class ViewHost(C.Structure):
    _fields_ = [
        ("T", c_int), ("N", c_int), ("action_kind", c_int), ("obs_dim", c_int), ("act_dim", c_int),
        ("hidden_dim", c_int), ("size", c_int), ("num_seqs", c_int), ("h0_rows", c_int),
        ("deficit", c_int), ("stale_steps", c_int), ("replayed_steps", c_int),
        ("snapshot_version", c_uint64), ("collect_wall_time", c_double),
        ("obs", P(c_float)), ("act_cont", P(c_float)), ("act_disc", P(c_int32)),
        ("log_prob", P(c_float)), ("value", P(c_float)), ("reward", P(c_float)),
        ("latency", P(c_float)), ("advantage", P(c_float)), ("returns", P(c_float)),
        ("done", P(C.c_uint8)), ("stale", P(C.c_uint8)), ("replayed", P(C.c_uint8)),
        ("env_index", P(c_int32)), ("seq_of_slot", P(c_int32)), ("step_in_episode", P(c_int32)),
        ("episode_index", P(c_int64)), ("version", P(c_uint64)),
        ("seqs", P(SeqDesc)), ("h0", P(c_float)),
        ("per_env_counts", P(c_int32)), ("env_bootstrap", P(c_float)),
        ("env_bootstrap_valid", P(C.c_uint8)),
    ]


class RolloutConfig(C.Structure):
    _fields_ = [("T", c_int), ("N", c_int), ("mode", c_int), ("action_kind", c_int),
                ("obs_dim", c_int), ("act_dim", c_int), ("hidden_dim", c_int)]


class StepBatch(C.Structure):
    _fields_ = [
        ("n", c_int), ("env_index", P(c_int32)), ("episode_index", P(c_int64)),
        ("step_in_episode", P(c_int32)), ("obs", P(c_float)), ("act_disc", P(c_int32)),
        ("act_cont", P(c_float)), ("log_prob", P(c_float)), ("value", P(c_float)),
        ("reward", P(c_float)), ("latency", P(c_float)), ("done", P(C.c_uint8)),
        ("h_before", P(c_float)), ("h_before_valid", P(C.c_uint8)),
        ("snapshot_version", P(c_uint64)),
    ]


class ModelConfig(C.Structure):
    _fields_ = [("obs_dim", c_int), ("encoder_dim", c_int), ("hidden_dim", c_int),
                ("action_kind", c_int), ("num_actions", c_int), ("act_dim", c_int)]


class EngineConfig(C.Structure):
    _fields_ = [("rollout", RolloutConfig), ("model", ModelConfig), ("seed", c_uint64)]


class RequestBatch(C.Structure):
    _fields_ = [("n", c_int), ("env_index", P(c_int32)), ("obs", P(c_float)), ("reward", P(c_float)),
                ("done", P(C.c_uint8)), ("first", P(C.c_uint8)), ("latency", P(c_float)),
                ("obs_episode", P(c_int64)), ("obs_step", P(c_int32))]


class BatchResult(C.Structure):
    _fields_ = [("n_dispatch", c_int), ("new_commits", c_int), ("closed_now", c_int), ("preempt_fired", c_int)]


class PPOConfig(C.Structure):
    _fields_ = [("gamma", c_double), ("gae_lambda", c_double), ("clip", c_double),
                ("epochs", c_int), ("minibatches", c_int), ("value_loss_coef", c_double),
                ("is_cap", c_double)]


class LossResult(C.Structure):
    _fields_ = [(n, c_double) for n in ("loss", "policy_loss", "value_loss", "mean_entropy",
                                         "ratio_sum", "clip_count", "w_sum", "w_max")] + [
        ("steps", c_int)]


class EntropyController(C.Structure):
    _fields_ = [(n, c_double) for n in ("alpha", "target", "lower", "upper", "lr")]


class TrainStats(C.Structure):
    _fields_ = [("update_index", c_int64), ("steps", c_int), ("fresh_steps", c_int),
                ("stale_steps", c_int)] + [
        (n, c_double) for n in ("loss", "policy_loss", "value_loss", "entropy", "entropy_loss",
                                "mean_ratio", "clip_fraction", "mean_is_weight", "max_is_weight",
                                "alpha", "lr")]


GradHook = C.CFUNCTYPE(c_int, C.c_void_p, C.c_void_p, c_int64, c_uint64)
EntropyHook = C.CFUNCTYPE(c_int, C.c_void_p, C.c_void_p, c_uint64)
SumI64 = C.CFUNCTYPE(c_int, C.c_void_p, P(c_int64), c_int)
MeanF64 = C.CFUNCTYPE(c_int, C.c_void_p, P(c_double), c_int)
AllgatherF64 = C.CFUNCTYPE(c_int, C.c_void_p, P(c_double), c_int, P(c_double))


class ReplicaComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("sum_i64", SumI64), ("mean_f64", MeanF64),
                ("allgather_f64", AllgatherF64), ("nranks", c_int), ("rank", c_int)]


class ReplicaConfig(C.Structure):
    _fields_ = [("T", c_int), ("N", c_int), ("preempt", c_int), ("per_replica_budget", c_int)]


class IterationResult(C.Structure):
    _fields_ = [("iteration", c_int64), ("rank", c_int), ("deficit", c_int), ("stale_steps", c_int),
                ("global_consumed_before", c_int64), ("global_fresh", c_int64), ("learn_time", c_double),
                ("mean_learn_time", c_double), ("next_threshold", c_int64),
                ("per_replica_threshold", c_int64), ("train", TrainStats)]


_SIGS = {
    "ver_version": (C.c_char_p, []),
    "ver_ctx_create": (c_int, [c_int, P(C.c_void_p)]),
    "ver_ctx_destroy": (c_int, [C.c_void_p]),
    "ver_ctx_synchronize": (c_int, [C.c_void_p]),
    "ver_ctx_stream": (c_int, [C.c_void_p, P(c_uint64)]),
    "ver_ctx_launch_count": (c_int, [C.c_void_p, P(c_int64), c_int]),
    "ver_ctx_set_precision": (c_int, [C.c_void_p, c_int]),
    "ver_ctx_set_tensor_cores": (c_int, [C.c_void_p, c_int]),
    "ver_nccl_unique_id": (c_int, [C.c_char_p]),
    "ver_ctx_init_nccl": (c_int, [C.c_void_p, C.c_char_p, c_int, c_int]),
    "ver_allreduce_sum_i64": (c_int, [C.c_void_p, P(c_int64), c_int]),
    "ver_allreduce_mean_f64": (c_int, [C.c_void_p, P(c_double), c_int]),
    "ver_allgather_f64": (c_int, [C.c_void_p, P(c_double), c_int, P(c_double)]),
    "ver_view_upload": (c_int, [C.c_void_p, P(ViewHost), P(C.c_void_p)]),
    "ver_view_info": (c_int, [C.c_void_p, P(ViewHost)]),
    "ver_view_download": (c_int, [C.c_void_p, P(ViewHost)]),
    "ver_view_clone": (c_int, [C.c_void_p, P(C.c_void_p)]),
    "ver_view_destroy": (c_int, [C.c_void_p]),
    "ver_view_restale": (c_int, [C.c_void_p, c_uint64]),
    "ver_rollout_create": (c_int, [C.c_void_p, P(RolloutConfig), P(C.c_void_p)]),
    "ver_rollout_destroy": (c_int, [C.c_void_p]),
    "ver_rollout_begin": (c_int, [C.c_void_p, c_uint64]),
    "ver_rollout_append": (c_int, [C.c_void_p, P(StepBatch), P(c_int32)]),
    "ver_rollout_force_close": (c_int, [C.c_void_p]),
    "ver_rollout_set_bootstrap": (c_int, [C.c_void_p, c_int, c_float]),
    "ver_rollout_set_bootstraps": (c_int, [C.c_void_p, c_int, P(c_int32), P(c_float)]),
    "ver_rollout_state": (c_int, [C.c_void_p, P(c_int), P(c_int), P(c_int)]),
    "ver_rollout_close": (c_int, [C.c_void_p, P(C.c_void_p)]),
    "ver_view_synth": (c_int, [C.c_void_p, P(c_int32), c_int, c_int, c_int, c_uint64, c_float, P(C.c_void_p)]),
    "ver_bench_gae_gather": (c_int, [C.c_void_p, c_double, c_double, c_int, c_uint64, c_int, P(c_float)]),
    "ver_backfill_stale": (c_int, [C.c_void_p, C.c_void_p, c_int]),
    "ver_compute_gae": (c_int, [C.c_void_p, c_double, c_double]),
    "ver_split_minibatches": (c_int, [C.c_void_p, c_int, c_uint64, P(C.c_void_p)]),
    "ver_split_in_order": (c_int, [C.c_void_p, c_int, P(c_int32), c_int, P(C.c_void_p)]),
    "ver_groups_count": (c_int, [C.c_void_p, P(c_int)]),
    "ver_groups_get": (c_int, [C.c_void_p, c_int, P(c_int), P(c_int), P(SeqDesc)]),
    "ver_groups_destroy": (c_int, [C.c_void_p]),
    "ver_pack": (c_int, [C.c_void_p, C.c_void_p, c_int, P(C.c_void_p)]),
    "ver_pack_seqs": (c_int, [C.c_void_p, P(SeqDesc), c_int, P(C.c_void_p)]),
    "ver_packed_info": (c_int, [C.c_void_p, P(c_int), P(c_int), P(c_int)]),
    "ver_packed_get": (c_int, [C.c_void_p, P(SeqDesc), P(c_int32), P(c_int32), P(c_int32), P(c_int32)]),
    "ver_packed_get_gathered": (c_int, [C.c_void_p, P(c_float), P(c_int32), P(c_float), P(c_float),
                                        P(c_float), P(c_float)]),
    "ver_packed_destroy": (c_int, [C.c_void_p]),
    "ver_param_count": (c_int, [P(ModelConfig), P(c_int64), P(c_int)]),
    "ver_param_tensor": (c_int, [P(ModelConfig), c_int, C.c_char_p, P(c_int), P(c_int), P(c_int64)]),
    "ver_params_init": (c_int, [P(ModelConfig), c_uint64, P(c_double)]),
    "ver_ppo_loss": (c_int, [C.c_void_p, P(ModelConfig), P(c_float), C.c_void_p, C.c_void_p,
                             P(PPOConfig), c_double, P(c_float), c_int, P(c_float), P(LossResult),
                             P(c_float), P(c_float)]),
    "ver_forward_packed": (c_int, [C.c_void_p, P(ModelConfig), P(c_float), c_int, P(c_float), P(c_int32),
                                   P(c_float), c_int, P(c_int32), P(c_int32), P(c_float), P(c_float),
                                   P(c_float), P(c_float)]),
    "ver_act": (c_int, [C.c_void_p, P(ModelConfig), P(c_float), c_int, P(c_float), P(c_float),
                        P(c_float), P(c_float), P(c_float)]),
    "ver_adam_step": (c_int, [C.c_void_p, c_int64, P(c_float), P(c_float), P(c_float), P(c_float),
                              P(c_int64), c_double]),
    "ver_cosine_lr": (c_double, [c_double, c_int64, c_int64]),
    "ver_learner_create": (c_int, [C.c_void_p, P(ModelConfig), P(c_float), P(PPOConfig),
                                   P(EntropyController), c_double, c_int64, c_uint64, P(C.c_void_p)]),
    "ver_learner_destroy": (c_int, [C.c_void_p]),
    "ver_learner_enable_allreduce": (c_int, [C.c_void_p, c_int]),
    "ver_learner_set_grad_hook": (c_int, [C.c_void_p, GradHook, C.c_void_p]),
    "ver_learner_set_entropy_hook": (c_int, [C.c_void_p, EntropyHook, C.c_void_p]),
    "ver_param_device_index": (c_int, [P(ModelConfig), P(c_int64)]),
    "ver_replica_create": (c_int, [C.c_void_p, C.c_void_p, P(ReplicaConfig), P(ReplicaComm), P(C.c_void_p)]),
    "ver_replica_destroy": (c_int, [C.c_void_p]),
    "ver_replica_attach_preempt": (c_int, [C.c_void_p, C.c_void_p]),
    "ver_replica_learn": (c_int, [C.c_void_p, C.c_void_p, c_double, c_int, P(IterationResult)]),
    "ver_replica_state": (c_int, [C.c_void_p, P(c_int64), P(c_int64), P(c_int)]),
    "ver_learner_update": (c_int, [C.c_void_p, C.c_void_p, P(TrainStats)]),
    "ver_learner_batch_h0": (c_int, [C.c_void_p, C.c_void_p, C.c_void_p, P(c_float)]),
    "ver_learner_get_params": (c_int, [C.c_void_p, P(c_float)]),
    "ver_learner_set_params": (c_int, [C.c_void_p, P(c_float)]),
    "ver_learner_get_adam": (c_int, [C.c_void_p, P(c_float), P(c_float), P(c_int64)]),
    "ver_learner_set_adam": (c_int, [C.c_void_p, P(c_float), P(c_float), c_int64]),
    "ver_learner_get_state": (c_int, [C.c_void_p, P(c_double), P(c_int64), P(c_int64)]),
    "ver_learner_set_state": (c_int, [C.c_void_p, c_double, c_int64, c_int64]),
    "ver_learner_last_timing": (c_int, [C.c_void_p, P(c_float), P(c_int)]),
    "ver_learner_last_timing_counts": (c_int, [C.c_void_p, P(c_int), P(c_int)]),
    "ver_learner_last_flop": (c_int, [C.c_void_p, P(C.c_double), P(c_int)]),
    "ver_debug_gemm": (c_int, [C.c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, P(c_float), c_int,
                               P(c_float), c_int, P(c_float), c_int]),
    "ver_debug_gemm_time": (c_int, [C.c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                    P(c_float)]),
    "ver_debug_gemm_prof": (c_int, [C.c_void_p, c_int, P(C.c_ulonglong)]),
    "ver_preempt_create": (c_int, [C.c_void_p, P(C.c_void_p)]),
    "ver_preempt_ipc_handle": (c_int, [C.c_void_p, P(C.c_uint8)]),
    "ver_preempt_open": (c_int, [C.c_void_p, P(C.c_uint8), P(C.c_void_p)]),
    "ver_preempt_destroy": (c_int, [C.c_void_p]),
    "ver_preempt_start": (c_int, [C.c_void_p, c_int64]),
    "ver_preempt_add": (c_int, [C.c_void_p, c_int64, P(c_int64), P(c_int)]),
    "ver_preempt_state": (c_int, [C.c_void_p, P(c_int64), P(c_int)]),
    "ver_preempt_create_nccl": (c_int, [C.c_void_p, P(C.c_void_p)]),
    "ver_preempt_tick": (c_int, [C.c_void_p, P(c_int64), P(c_int)]),
    "ver_view_dump_jsonl": (c_int, [C.c_void_p, C.c_char_p]),
    "ver_view_load_jsonl": (c_int, [C.c_void_p, C.c_char_p, P(C.c_void_p)]),
    "ver_learner_save_checkpoint": (c_int, [C.c_void_p, C.c_char_p]),
    "ver_checkpoint_model_config": (c_int, [C.c_char_p, P(ModelConfig)]),
    "ver_learner_load_checkpoint": (c_int, [C.c_void_p, C.c_char_p]),
    "ver_engine_create": (c_int, [C.c_void_p, P(EngineConfig), P(c_float), c_uint64, P(C.c_void_p)]),
    "ver_engine_destroy": (c_int, [C.c_void_p]),
    "ver_engine_set_snapshot": (c_int, [C.c_void_p, P(c_float), c_uint64]),
    "ver_engine_set_snapshot_learner": (c_int, [C.c_void_p, C.c_void_p, c_uint64]),
    "ver_engine_begin_rollout": (c_int, [C.c_void_p, P(BatchResult), P(c_int32), P(c_int32), P(c_float)]),
    "ver_engine_process_batch": (c_int, [C.c_void_p, P(RequestBatch), P(BatchResult), P(c_int32), P(c_int32),
                                         P(c_float)]),
    "ver_engine_force_close": (c_int, [C.c_void_p]),
    "ver_engine_attach_preempt": (c_int, [C.c_void_p, C.c_void_p]),
    "ver_engine_finalize_bootstraps": (c_int, [C.c_void_p]),
    "ver_engine_close": (c_int, [C.c_void_p, P(C.c_void_p)]),
    "ver_engine_state": (c_int, [C.c_void_p, P(c_int), P(c_int), P(c_int), P(c_int), P(c_int)]),
    "ver_engine_hidden": (c_int, [C.c_void_p, P(c_float)]),
    "ver_estimate_time": (c_int, [C.c_void_p, P(c_double), c_int, c_int64, c_int64, P(c_double)]),
    "ver_optimal_preempt_steps": (c_int, [C.c_void_p, P(c_double), c_int, c_double, c_int64,
                                          P(c_int64)]),
}

EXPORTS = tuple(_SIGS) + ("ver_last_error",)

_lib = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libver_b200.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is missing: run `python -m paper_2210_05064_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    lib.ver_last_error.restype = C.c_char_p
    lib.ver_last_error.argtypes = []
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
