"""Overlapped collection and learning (the reference's
overlap mode, bench.cpp:129-160, Appendix E of the paper) on one GPU.

The inference engine and the learner run on separate contexts (CUDA streams)
driven by separate host threads: while the learner updates on rollout k, the
engine collects rollout k+1 with the pre-update snapshot.  The learner then
publishes its parameters to the engine device to device, and rollout k+1 is
restaled against the learner's version before its update (rollout.cpp:15-22),
so its lagged steps are marked stale (the IS cap of the loss handles them).

`collect(engine)` is the caller's environment loop: it drives
engine.begin_rollout / process_batch (or process_arrays) until the rollout
closes and returns engine.close() (after finalize_bootstraps)."""
from __future__ import annotations

import threading
from typing import Callable

from . import api as V


class OverlappedTrainer:
    def __init__(self, engine: V.InferenceEngine, learner: V.Learner,
                 collect: Callable[[V.InferenceEngine], V.RolloutView]):
        if engine.ctx is learner.ctx:
            raise V.ConfigError("overlap: the engine and the learner need separate contexts (streams)")
        self.engine, self.learner, self.collect = engine, learner, collect
        self.pending: V.RolloutView | None = None
        self.version = 0

    def prime(self):
        """Collect rollout 0 with snapshot 0 (bench.cpp:131-134)."""
        self.pending = self.collect(self.engine)
        self.engine.ctx.synchronize()

    def iteration(self, read_stats: bool = True) -> V.TrainStats | None:
        """One overlapped iteration: collect k+1 (snapshot k) while updating on k."""
        if self.pending is None:
            self.prime()
        view = self.pending
        view.restale(self.version)  # marks lagged data (overlap mode) for the IS cap
        self.engine.ctx.synchronize()  # the view (engine stream) is complete before the learner reads it
        box: dict = {}

        def run():
            try:
                box["view"] = self.collect(self.engine)
                self.engine.ctx.synchronize()
            except BaseException as e:  # re-raised on the caller's thread
                box["err"] = e

        th = threading.Thread(target=run)
        th.start()
        stats = self.learner.update(view, read_stats=read_stats)
        self.learner.ctx.synchronize()
        th.join()
        if "err" in box:
            raise box["err"]
        self.version += 1
        self.engine.set_snapshot_from(self.learner, self.version)
        self.pending = box["view"]
        return stats
