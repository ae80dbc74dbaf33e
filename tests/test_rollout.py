"""Port of the reference's tests/test_rollout.cpp (rollout store, compaction,
backfill) run on both the oracle and the device store."""
import numpy as np
import pytest

from backends import BACKENDS, make_backend, protocol_errors
from helpers import rec, records
from paper_2210_05064_b200.rng import CounterRng

FIXED, VARIABLE = 0, 1


@pytest.fixture(params=BACKENDS)
def be(request):
    return make_backend(request.param)


def app(buf, *rs):
    return buf.append(records(list(rs)))


def test_variable_mode_accepts_any_mix(be):  # test_rollout.cpp:44-67
    buf = be.rollout(4, 4, VARIABLE)
    buf.begin_rollout(1)
    counts = [6, 2, 4, 4]
    t = [0] * 4
    left = list(counts)
    committed = 0
    while committed < 16:
        for e in range(4):
            if left[e] > 0:
                assert app(buf, rec(e, 0, t[e], False))[0] == 0
                t[e] += 1
                left[e] -= 1
                committed += 1
                if committed == 16:
                    break
    assert buf.committed() == 16
    assert not buf.open()
    v = be.host(buf.close_rollout())
    assert v.size == 16
    assert list(v.per_env_counts) == counts


def test_fixed_mode_cap(be):  # test_rollout.cpp:69-82
    buf = be.rollout(4, 2, FIXED)
    buf.begin_rollout(1)
    for t in range(4):
        assert app(buf, rec(0, 0, t, False))[0] == 0
    assert app(buf, rec(0, 0, 4, False))[0] == 1
    assert buf.committed() == 4
    for t in range(4):
        app(buf, rec(1, 0, t, False))
    assert not buf.open()
    v = be.host(buf.close_rollout())
    assert list(v.per_env_counts) == [4, 4]
    buf.begin_rollout(2)
    assert app(buf, rec(0, 0, 4, False))[0] == 0


def test_carryover(be):  # test_rollout.cpp:84-114
    buf = be.rollout(2, 2, VARIABLE)
    buf.begin_rollout(1)
    for t in range(3):
        app(buf, rec(0, 0, t, False))
    app(buf, rec(1, 0, 0, False))
    assert not buf.open()
    assert app(buf, rec(1, 0, 1, False, reward=7.0))[0] == 1
    assert buf.carryover_count() == 1
    with pytest.raises(protocol_errors()):
        app(buf, rec(1, 0, 2, False))
    buf.close_rollout()
    buf.begin_rollout(2)
    assert buf.committed() == 1
    assert buf.carryover_count() == 0
    for t in range(3):
        app(buf, rec(0, 1, t, False))
    v = be.host(buf.close_rollout())
    found = False
    for i in range(v.size):
        if v.env_index[i] == 1 and v.step_in_episode[i] == 1:
            assert v.reward[i] == pytest.approx(7.0)
            found = True
    assert found


def test_sequence_boundaries(be):  # test_rollout.cpp:116-131
    buf = be.rollout(3, 2, VARIABLE)
    buf.begin_rollout(1)
    app(buf, rec(0, 0, 0, False), rec(0, 0, 1, True), rec(0, 1, 0, False), rec(1, 0, 0, False),
        rec(1, 0, 1, False), rec(1, 0, 2, False))
    v = be.host(buf.close_rollout())
    assert v.num_seqs == 3
    assert list(v.seqs[:, 2]) == [2, 1, 3]


def test_k_equals_contributing_envs(be):  # test_rollout.cpp:133-140
    buf = be.rollout(2, 3, VARIABLE)
    buf.begin_rollout(1)
    for e in range(3):
        for t in range(2):
            app(buf, rec(e, 0, t, False))
    v = be.host(buf.close_rollout())
    assert v.num_seqs == 3


def test_boundary_property(be):  # test_rollout.cpp:142-174
    rng = CounterRng(17)
    for trial in range(50):
        buf = be.rollout(8, 3, VARIABLE)
        buf.begin_rollout(1)
        t = [0, 0, 0]
        ep = [0, 0, 0]
        while buf.open():
            e = int(rng.uniform_int(3))
            done = rng.uniform() < 0.2
            app(buf, rec(e, ep[e], t[e], done))
            if done:
                ep[e] += 1
                t[e] = 0
            else:
                t[e] += 1
        v = be.host(buf.close_rollout())
        for i in range(1, v.size):
            if v.env_index[i] != v.env_index[i - 1]:
                continue
            changed = v.seq_of_slot[i] != v.seq_of_slot[i - 1]
            assert changed == bool(v.done[i - 1])
        for i in range(v.size):
            if i == 0 or v.env_index[i] != v.env_index[i - 1]:
                assert v.seqs[v.seq_of_slot[i], 3] == i


def test_empty_close_throws(be):  # test_rollout.cpp:176-181
    buf = be.rollout(2, 2, VARIABLE)
    buf.begin_rollout(1)
    buf.force_close()
    with pytest.raises(protocol_errors()):
        buf.close_rollout()


def _prev_and_preempted(be):
    buf = be.rollout(8, 2, VARIABLE)
    buf.begin_rollout(1)
    t = [0, 0]
    while buf.open():
        e = buf.committed() % 2
        app(buf, rec(e, 0, t[e], False))
        t[e] += 1
    prev = buf.close_rollout()
    buf.begin_rollout(2)
    for i in range(10):
        app(buf, rec(i % 2, 1, i // 2, False))
    buf.force_close()
    v = buf.close_rollout()
    return prev, v


def test_preempted_backfill(be):  # test_rollout.cpp:183-216
    prev, v = _prev_and_preempted(be)
    assert be.host(prev).size == 16
    assert be.host(v).deficit == 6
    w0 = be.clone(v)
    be.backfill(v, prev, be.host(v).deficit)
    hv = be.host(v)
    assert hv.size == 16
    assert hv.stale_steps == 6
    assert int(hv.stale.sum()) == 6
    # deficit zero leaves the view unchanged
    w = be.clone(v)
    be.backfill(w, prev, 0)
    assert be.host(w).size == hv.size and be.host(w).stale_steps == hv.stale_steps
    # deficit beyond the previous rollout size throws
    with pytest.raises(protocol_errors()):
        be.backfill(w0, prev, be.host(prev).size + 1)


def test_conservation_with_carryover(be):  # test_rollout.cpp:218-240
    buf = be.rollout(4, 2, VARIABLE)
    produced = committed_total = 0
    t = [0, 0]
    rng = CounterRng(3)
    for r in range(5):
        buf.begin_rollout(r + 1)
        while buf.open():
            e = int(rng.uniform_int(2))
            app(buf, rec(e, 0, t[e], False))
            t[e] += 1
            produced += 1
        e = int(rng.uniform_int(2))
        app(buf, rec(e, 0, t[e], False))
        t[e] += 1
        produced += 1
        committed_total += be.host(buf.close_rollout()).size
    assert committed_total == 5 * 8
    assert produced == committed_total + buf.carryover_count()


def test_h0_rows_and_descriptors(be):
    """h0 row of each sequence = h_before of its first record, zeros at episode
    restarts inside the rollout when absent (rollout.cpp:155-157)."""
    buf = be.rollout(3, 2, VARIABLE)
    buf.begin_rollout(9)
    rs = [rec(0, 0, 0, False, 0.5), rec(0, 0, 1, True, 1.0), rec(1, 0, 0, False),
          rec(1, 0, 1, False), rec(0, 1, 0, False), rec(1, 0, 2, False)]
    r = records(rs)
    r.h_before_valid = np.array([1, 1, 1, 1, 0, 1], np.uint8)
    buf.append(r)
    buf.set_bootstrap(0, 0.25)
    buf.set_bootstrap(1, -0.5)
    v = be.host(buf.close_rollout())
    assert v.num_seqs == 3
    np.testing.assert_allclose(v.h0[0], 0.0)          # env 0 -> 0.01*0
    np.testing.assert_allclose(v.h0[1], 0.0)          # absent -> zeros
    np.testing.assert_allclose(v.h0[2], 0.01, rtol=1e-6)  # env 1
    assert list(v.seqs[:, 1]) == [0, 0, 1]
    assert list(v.seqs[:, 3]) == [0, 2, 3]
    assert v.env_bootstrap[0] == pytest.approx(0.25)
    assert list(v.env_bootstrap_valid) == [1, 1]
    assert v.snapshot_version == 9
