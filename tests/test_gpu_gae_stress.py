"""GAE edge cases of the warp-tile scan (csrc/gae.cu: 512-slot tiles + a
128-slot halo row, look-back only across reset-free halos) vs the oracle's
compute_gae (learner.cpp:11-41) and an independent float64 recursion:

* envs with no fresh slot (tail slots read their env directly);
* segments longer than several tiles (reset-free halos: the look-back chain,
  gamma * lambda close to 1);
* array sizes around multiples of the tile and of tile + halo (partial top
  tile, halos read from global memory, 4-slot tails);
* resets exactly on the halo / bottom-row boundaries.

Bar: |gpu - ref| <= 1e-5 * max(1, |ref|)."""
from dataclasses import replace

import numpy as np
import pytest

from test_gpu_parity import assert_close
from test_gpu_ragged import gae_ref

pytestmark = pytest.mark.gpu


def _both(wl, T, N, H, force=False):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    g = V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H)
    o = O.Rollout(T, N, 1, 0, 2, 0, H)
    for buf in (g, o):
        synth.fill_buffer(buf, wl)
        if force:
            buf.force_close()
    return g.close_rollout(), o.close_rollout()


def _drop_envs(wl, envs):
    import paper_2210_05064_b200 as V
    keep = ~np.isin(np.asarray(wl.records.env_index), envs)
    recs = V.StepRecords(**{k: (None if v is None else np.asarray(v)[keep])
                            for k, v in wl.records.__dict__.items()})
    valid = np.asarray(wl.bootstrap_valid).copy()
    valid[envs] = 0
    return replace(wl, records=recs, bootstrap_valid=valid)


def test_gae_envs_without_fresh_slots():
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    T, N, H = 64, 96, 4
    wl = _drop_envs(synth.make_workload(T, N, hidden_dim=H, seed=21), [0, 5, 6, 7, 40, 95])
    vg, vo = _both(wl, T, N, H, force=True)
    hv = vg.to_host()
    assert hv.per_env_counts[[0, 5, 6, 7, 40, 95]].sum() == 0
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    hg, ho = vg.to_host(), vo.to_host()
    assert_close(hg.advantage, ho.advantage, what="A")
    assert_close(hg.returns, ho.returns, what="R")


@pytest.mark.parametrize("gl", [(0.999, 0.999), (1.0, 1.0), (0.99, 0.95)])
def test_gae_segments_longer_than_a_tile(gl):
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from paper_2210_05064_b200 import synth
    T, N, H = 3000, 4, 4
    wl = synth.make_workload(T, N, hidden_dim=H, seed=22, p_done=2e-4)
    vg, vo = _both(wl, T, N, H)
    assert int(np.max(vg.to_host().per_env_counts)) > 2048
    V.compute_gae(vg, *gl)
    O.compute_gae(vo, *gl)
    hg, ho = vg.to_host(), vo.to_host()
    scale = max(1.0, float(np.abs(ho.advantage).max()))
    # values grow to O(segment length) at gamma = lambda = 1: scale the bar by the magnitude
    assert np.abs(hg.advantage - ho.advantage).max() <= 1e-5 * scale
    assert np.abs(hg.returns - ho.returns).max() <= 1e-5 * scale


@pytest.mark.parametrize("S", [1, 3, 512, 513, 516, 640, 644, 645, 1023, 1024 + 131, 2048, 2049, 2052,
                               3 * 2048 - 1, 3 * 2048 + 3, 5 * 2048 + 7])
def test_gae_tile_boundaries(S):
    import paper_2210_05064_b200 as V
    rng = np.random.default_rng(S)
    lens = rng.integers(1, 400, size=S)
    lens = lens[np.cumsum(lens) <= S]
    if lens.sum() < S:
        lens = np.append(lens, S - lens.sum())
    view = V.view_synth(lens.astype(np.int32), seed=S, p_done=1.0 / 600)
    V.compute_gae(view, 0.99, 0.97)
    hv = view.to_host()
    assert hv.size == S
    ref = gae_ref(hv, 0.99, 0.97)
    err = np.abs(hv.advantage - ref) / np.maximum(1.0, np.abs(ref))
    assert err.max() <= 1e-5


@pytest.mark.parametrize("period", [128, 129, 511, 512, 640, 700])
def test_gae_reset_at_tile_and_halo_boundaries(period):
    """Envs of exactly `period` slots without dones: the only resets are env
    tails, placed on / next to the 128-slot row, 512-slot tile and halo
    boundaries, so tiles alternate between local carries and look-backs."""
    import paper_2210_05064_b200 as V
    S = 40 * 512 + 17
    lens = np.full(S // period, period, np.int64)
    if lens.sum() < S:
        lens = np.append(lens, S - lens.sum())
    view = V.view_synth(lens.astype(np.int32), seed=period, p_done=0.0)
    V.compute_gae(view, 0.999, 0.999)
    hv = view.to_host()
    ref = gae_ref(hv, 0.999, 0.999)
    err = np.abs(hv.advantage - ref) / np.maximum(1.0, np.abs(ref))
    assert err.max() <= 1e-5
