"""One interface over the two implementations the ported reference tests run on.

``oracle``: the CPU double restatement (checker, pinned by these tests).
``gpu``: libver_b200.so through the C-ABI (the product).
"""
from __future__ import annotations

import numpy as np
import pytest


class GroupView:
    def __init__(self, seqs: np.ndarray, total: int):
        self.seqs = np.asarray(seqs, np.int32).reshape(-1, 8)
        self.total_steps = total

    # field accessors by name (SequenceDescriptor, rollout.hpp:19-28)
    def col(self, name: str) -> np.ndarray:
        from paper_2210_05064_b200.hostview import SEQ_FIELDS
        return self.seqs[:, SEQ_FIELDS.index(name)]


class OracleBackend:
    name = "oracle"

    def __init__(self):
        from oracle import oracle as O
        self.O = O

    def rollout(self, T, N, mode=1, action_kind=0, obs_dim=2, act_dim=0, hidden_dim=3):
        O = self.O

        class R:
            def __init__(s):
                s.r = O.Rollout(T, N, mode, action_kind, obs_dim, act_dim, hidden_dim)

            def begin_rollout(s, v):
                s.r.begin_rollout(v)

            def append(s, recs):
                return s.r.append_steps(recs)

            def force_close(s):
                s.r.force_close()

            def set_bootstrap(s, e, v):
                s.r.set_bootstrap(e, v)

            def open(s):
                return bool(s.r.state()[0])

            def committed(s):
                return s.r.state()[1]

            def carryover_count(s):
                return s.r.state()[2]

            def close_rollout(s):
                return s.r.close_rollout()

        return R()

    def upload(self, hv):
        return self.O.View.from_host(hv)

    def host(self, view):
        return view.to_host()

    def clone(self, view):
        return view.clone()

    def backfill(self, view, prev, deficit):
        self.O.backfill_stale(view, prev, deficit)

    def gae(self, view, g, l):
        self.O.compute_gae(view, g, l)

    def split(self, view, B, seed):
        return [GroupView(s, t) for s, t in self.O.split_minibatches(view, B, seed).groups()]

    def split_in_order(self, view, B, order):
        return [GroupView(s, t) for s, t in self.O.split_in_order(view, B, order).groups()]

    def pack(self, view, group: GroupView):
        return self.O.pack(group.seqs)

    def estimate_time(self, tau, smax, s):
        return self.O.estimate_time(tau, smax, s)

    def optimal_preempt_steps(self, tau, lt, smax):
        return self.O.optimal_preempt_steps(tau, lt, smax)

    protocol_error = None  # set below


class GpuBackend:
    name = "gpu"

    def __init__(self):
        import paper_2210_05064_b200 as V
        self.V = V

    def rollout(self, T, N, mode=1, action_kind=0, obs_dim=2, act_dim=0, hidden_dim=3):
        V = self.V

        class R:
            def __init__(s):
                s.r = V.RolloutBuffer(T, N, mode, action_kind, obs_dim, act_dim, hidden_dim)

            def begin_rollout(s, v):
                s.r.begin_rollout(v)

            def append(s, recs):
                return s.r.append_steps(recs)

            def force_close(s):
                s.r.force_close()

            def set_bootstrap(s, e, v):
                s.r.set_bootstrap(e, v)

            def open(s):
                return s.r.open()

            def committed(s):
                return s.r.committed()

            def carryover_count(s):
                return s.r.carryover_count()

            def close_rollout(s):
                return s.r.close_rollout()

        return R()

    def upload(self, hv):
        return self.V.RolloutView.from_host(hv)

    def host(self, view):
        return view.to_host()

    def clone(self, view):
        return view.clone()

    def backfill(self, view, prev, deficit):
        self.V.backfill_stale(view, prev, deficit)

    def gae(self, view, g, l):
        self.V.compute_gae(view, g, l)

    def split(self, view, B, seed):
        return [GroupView(g.seqs, g.total_steps) for g in self.V.split_minibatches(view, B, seed)]

    def split_in_order(self, view, B, order):
        return [GroupView(g.seqs, g.total_steps) for g in self.V.split_in_order(view, B, order)]

    def pack(self, view, group: GroupView):
        b = self.V.pack(view, self.V.SequenceGroup(group.seqs, group.total_steps))
        return b

    def estimate_time(self, tau, smax, s):
        return self.V.estimate_time(tau, smax, s)

    def optimal_preempt_steps(self, tau, lt, smax):
        return self.V.optimal_preempt_steps(tau, lt, smax)


def protocol_errors():
    from oracle.oracle import OracleProtocolError
    from paper_2210_05064_b200.api import ProtocolError
    return (OracleProtocolError, ProtocolError)


BACKENDS = [pytest.param("oracle", id="oracle"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


def make_backend(name: str):
    return OracleBackend() if name == "oracle" else GpuBackend()
