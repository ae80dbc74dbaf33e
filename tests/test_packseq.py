"""Port of the reference's tests/test_packseq.cpp (split + pack), on the oracle
and on the device sampler; plus bit-exact device-vs-oracle index parity."""
import numpy as np
import pytest

from backends import BACKENDS, GroupView, make_backend, protocol_errors
from helpers import make_view, random_lengths
from paper_2210_05064_b200.rng import CounterRng


@pytest.fixture(params=BACKENDS)
def be(request):
    return make_backend(request.param)


def test_greedy_fill_splits(be):  # test_packseq.cpp:14-35
    v = be.upload(make_view([2, 1, 3, 6, 4]))
    g = be.split_in_order(v, 2, [0, 1, 2, 3, 4])
    assert len(g) == 2
    assert g[0].total_steps == 8 and g[1].total_steps == 8
    assert list(g[0].col("length")) == [2, 1, 3, 2]
    assert g[0].col("skip")[3] == 0
    assert list(g[1].col("length")) == [4, 4]
    assert g[1].col("skip")[0] == 2
    assert g[1].col("seq_id")[0] == g[0].col("seq_id")[3]
    assert g[1].col("parent_start_offset")[0] == g[0].col("start_offset")[3]


def test_b1_one_minibatch(be):  # test_packseq.cpp:37-43
    v = be.upload(make_view([3, 5, 2]))
    g = be.split(v, 1, 7)
    assert len(g) == 1 and g[0].total_steps == 10 and len(g[0].seqs) == 3


def test_equal_length_degenerate(be):  # test_packseq.cpp:45-53
    v = be.upload(make_view([4, 4, 4, 4], 2, 4, 4, 4))
    g = be.split(v, 4, 3)
    assert len(g) == 4
    for x in g:
        assert x.total_steps == 4 and len(x.seqs) == 1


def test_non_divisor_rejected(be):  # test_packseq.cpp:55-58
    v = be.upload(make_view([4, 4], 2, 4, 4, 2))
    with pytest.raises(protocol_errors()):
        be.split(v, 3, 0)


def test_pack_layout_321(be):  # test_packseq.cpp:60-70
    hv = make_view([3, 2, 1])
    v = be.upload(hv)
    b = be.pack(v, GroupView(hv.seqs, hv.size))
    assert list(b.batch_sizes) == [3, 2, 1]
    assert b.total_steps == 6
    assert hv.obs[b.slots[0], 0] == 0
    assert hv.obs[b.slots[1], 0] == 3
    assert hv.obs[b.slots[2], 0] == 5


def test_pack_single_and_equal(be):  # test_packseq.cpp:72-80
    h1 = make_view([5])
    b1 = be.pack(be.upload(h1), GroupView(h1.seqs, 5))
    assert list(b1.batch_sizes) == [1] * 5
    h2 = make_view([4, 4])
    b2 = be.pack(be.upload(h2), GroupView(h2.seqs, 8))
    assert list(b2.batch_sizes) == [2] * 4


def test_pack_rejects_empty(be):  # test_packseq.cpp:82-85
    h = make_view([2])
    with pytest.raises(protocol_errors()):
        be.pack(be.upload(h), GroupView(np.zeros((0, 8), np.int32), 0))


def _unpack(b):
    seqs, s2g, offs, slots = b.seqs, b.sorted_to_group, b.offsets, b.slots
    out = [None] * len(seqs)
    for j in range(len(seqs)):
        out[s2g[j]] = [int(slots[offs[t] + j]) for t in range(int(seqs[j][2]))]
    return out


def test_property_roundtrip(be):  # test_packseq.cpp:87-125 (200 trials)
    rng = CounterRng(99)
    for trial in range(200):
        T, N, B = 8, 4, 2
        lengths = random_lengths(T * N, T, rng)
        v = be.upload(make_view(lengths, 2, 4, T, N))
        groups = be.split(v, B, trial)
        assert len(groups) == B
        seen = set()
        for g in groups:
            assert g.total_steps == T * N // B
            b = be.pack(v, g)
            assert b.total_steps == g.total_steps
            bs = list(b.batch_sizes)
            assert all(bs[t] <= bs[t - 1] for t in range(1, len(bs)))
            assert sum(bs) == b.total_steps
            un = _unpack(b)
            assert len(un) == len(g.seqs)
            for s in range(len(g.seqs)):
                assert len(un[s]) == g.seqs[s][2]
                assert un[s] == [int(g.seqs[s][3]) + t for t in range(int(g.seqs[s][2]))]
            for slot in b.slots:
                assert int(slot) not in seen
                seen.add(int(slot))
            for j in range(len(b.seqs)):
                assert b.seqs[j][0] == g.seqs[b.sorted_to_group[j]][0]
        assert len(seen) == T * N


def test_epoch_permutations_reproducible(be):  # test_learner.cpp:322-336
    v = be.upload(make_view([4, 4, 4, 4], 2, 4, 4, 4))

    def fp(gs):
        return [int(s[0]) for g in gs for s in g.seqs]

    assert fp(be.split(v, 2, 100)) == fp(be.split(v, 2, 100))
    assert fp(be.split(v, 2, 100)) != fp(be.split(v, 2, 101))


@pytest.mark.gpu
def test_device_split_pack_bitexact_vs_oracle():
    """Device deal + pack == oracle (libstdc++ shuffle, greedy fill, stable sort)
    bit for bit on ragged views, including uneven B and long straddlers."""
    o, g = make_backend("oracle"), make_backend("gpu")
    rng = CounterRng(5)
    for trial in range(60):
        N = 1 + int(rng.uniform_int(40))
        T = 1 + int(rng.uniform_int(64))
        lengths = random_lengths(T * N, 1 + int(rng.uniform_int(3 * T)), rng)
        hv = make_view(lengths, 2, 4, T, N)
        vo, vg = o.upload(hv), g.upload(hv)
        for B in (1, 2, 3, 5):
            if (T * N) % B:
                continue
            seed = rng.next_u64()
            go, gg = o.split(vo, B, seed), g.split(vg, B, seed)
            assert len(go) == len(gg)
            for a, b in zip(go, gg):
                np.testing.assert_array_equal(a.seqs, b.seqs)
                assert a.total_steps == b.total_steps
                if len(a.seqs) == 0:
                    continue
                pa, pb = o.pack(vo, a), g.pack(vg, b)
                np.testing.assert_array_equal(pa.seqs, pb.seqs)
                np.testing.assert_array_equal(pa.sorted_to_group, pb.sorted_to_group)
                np.testing.assert_array_equal(pa.batch_sizes, pb.batch_sizes)
                np.testing.assert_array_equal(pa.offsets, pb.offsets)
                np.testing.assert_array_equal(pa.slots, pb.slots)
