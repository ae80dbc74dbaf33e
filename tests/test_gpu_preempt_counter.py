"""Joint preemption counter (csrc/coordinator.cu, SURVEY §8(f) row 2;
PreemptCoordinator, distributed.hpp:95-128) across two processes on one device:
replica 0 owns the counter and exports its IPC handle, replica 1 opens it;
both add steps concurrently; exactly one add fires, at the first total >= the
threshold, and a threshold <= 0 never fires (per-replica-budget ablation)."""
import os
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CHILD = textwrap.dedent("""
    import sys, time
    sys.path.insert(0, {root!r})
    import paper_2210_05064_b200 as V
    h = bytes.fromhex(open({hpath!r}).read().strip())
    c = V.PreemptCounter(handle=h)
    fired = []
    for i in range({n}):
        t, f = c.add_steps({step})
        if f:
            fired.append(t)
    print("child", len(fired), *fired)
""")


def test_counter_fires_once_across_processes(tmp_path):
    import paper_2210_05064_b200 as V
    own = V.PreemptCounter()
    hpath = tmp_path / "h.txt"
    hpath.write_text(own.ipc_handle().hex())
    for threshold, n, step in ((1000, 400, 3), (0, 200, 5)):
        own.start_iteration(threshold)
        child = subprocess.Popen([sys.executable, "-c", CHILD.format(root=str(ROOT), hpath=str(hpath), n=n,
                                                                      step=step)],
                                 stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
        mine = []
        for i in range(n):
            t, f = own.add_steps(2)
            if f:
                mine.append(t)
        out, err = child.communicate(timeout=300)
        assert child.returncode == 0, err
        parts = out.split()
        theirs = [int(x) for x in parts[2:]] if parts[0] == "child" else []
        total, fired = own.state()
        if threshold > 0:
            assert total == n * 2 + n * step
            assert fired and len(mine) + len(theirs) == 1
            t_fire = (mine + theirs)[0]
            assert threshold <= t_fire < threshold + max(2, step)
        else:  # disabled: add_steps returns without counting (distributed.hpp:111)
            assert total == 0 and not fired and not mine and not theirs
