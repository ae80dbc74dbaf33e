"""Parity of the GRU recurrence paths that run at production sizes (H = 256 /
512) against the oracle's full Learner::update (learner.cpp:132-193):

* the persistent K-split kernels (gru_fwd_ks / gru_bwd_ks),
* the single-cluster tail kernels for the last short timesteps (H = 512),
* the tcgen05 path for timesteps with many rows: the persistent split-K step
  kernel (stepgemm.cu), single CTAs and CTA pairs, the latter with the forward
  gates fused into the GEMM epilogue,

each forced by the row thresholds (VER_REC_BIG_FWD / _BWD, VER_REC_TAIL_*),
which the library reads at every launch.

Bars: loss statistics and gradients within 1e-5 * max(1, |oracle|) (and
normwise 1e-5).  Parameters after an update: Adam's first step moves every
parameter by lr * g / (|g| + eps), i.e. by +-lr whatever |g| is, so a gradient
component that is zero up to fp32 rounding can move by a visible fraction of
lr; at H = 512 a handful of the 1.8M parameters sit above 1e-5.  The update
test therefore asserts 1e-5 on >= 99.99% of the parameters and 1e-4 on all."""
import os

import numpy as np
import pytest

from test_gpu_parity import _learner_pair, assert_close, close_both

pytestmark = pytest.mark.gpu

PATHS = {
    # K-split kernels only
    "ks": {"VER_REC_TAIL": "0", "VER_REC_BIG_FWD": "100000", "VER_REC_BIG_BWD": "100000"},
    # big steps (>= 6 rows) in the split-K tcgen05 step kernel (stepgemm.cu), K-split
    # for 5, cluster tail for <= 4 / <= 3 (the defaults)
    "big+ks+tail": {"VER_REC_TAIL": "1", "VER_REC_BIG_FWD": "6", "VER_REC_BIG_BWD": "6"},
    # big steps (>= 6 rows) on CTA pairs (the C3 path) with every forward step
    # split-K free and its gates in the GEMM epilogue, consecutive steps chained
    # per row tile instead of by a grid barrier (VER_REC_FUSE_ALL forces what only
    # >= ~2,300-row steps reach naturally)
    "pair+fused": {"VER_REC_TAIL": "1", "VER_REC_BIG_FWD": "6", "VER_REC_BIG_BWD": "6",
                   "VER_REC_PAIR_ROWS": "6", "VER_REC_FUSE_ALL": "1"},
    # cluster tail for everything it can take, K-split for the rest
    "tail": {"VER_REC_TAIL": "1", "VER_REC_TAIL_FWD": "8", "VER_REC_TAIL_BWD": "8",
             "VER_REC_BIG_FWD": "100000", "VER_REC_BIG_BWD": "100000"},
}


@pytest.fixture
def env_paths(request):
    keys = set().union(*PATHS.values())
    saved = {k: os.environ.get(k) for k in keys}
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update(PATHS[request.param])
    yield request.param
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("env_paths", list(PATHS), indirect=True)
@pytest.mark.parametrize("H", [256, 512])
def test_update_parity_recurrence_paths(env_paths, H):
    T, N, epochs, B = 16, 24, 1, 2
    cfg, lg, lo = _learner_pair(H, H, epochs, B)
    vg, vo, _ = close_both(T, N, H, seed=31)
    sg = lg.update(vg)
    so = lo.update(vo)
    for k in ("loss", "policy_loss", "value_loss", "entropy", "mean_ratio", "alpha"):
        assert abs(getattr(sg, k) - so[k]) <= 1e-5 * max(1.0, abs(so[k])), (env_paths, k)
    pg, po = np.asarray(lg.params(), np.float64), np.asarray(lo.params(), np.float64)
    err = np.abs(pg - po) / np.maximum(1.0, np.abs(po))
    assert err.max() <= 1e-4, (env_paths, err.max())
    assert np.mean(err > 1e-5) <= 1e-4, (env_paths, int(np.sum(err > 1e-5)))
    m, _, _ = lg.adam()
    mo, _, _ = lo.adam()
    assert_close(m, mo, what=f"adam m ({env_paths}, H={H})")


@pytest.mark.parametrize("env_paths", list(PATHS), indirect=True)
@pytest.mark.parametrize("H", [256, 512])
def test_loss_gradient_parity_recurrence_paths(env_paths, H):
    """ppo_loss (forward, fused loss, backward through every recurrence path)
    vs the oracle on one packed minibatch of a C2-like view."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from test_gpu_parity import _model
    cfg = _model(H, H)
    p = O.params_init(cfg, O.mix(3, 0x9A9A)).astype(np.float32).astype(np.float64)
    vg, vo, _ = close_both(16, 24, H, seed=33)
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    hv = vo.to_host()
    bo = O.pack(hv.seqs)
    bg = V.pack(vg, V.SequenceGroup(hv.seqs))
    h0 = np.stack([hv.h0[s[4]] for s in bo.seqs])
    ro = O.ppo_loss(cfg, p, vo, bo, V.PPOConfig(), 0.01, h0, True)
    rg = V.ppo_loss(cfg, p, vg, bg, V.PPOConfig(), 0.01, h0, True)
    assert abs(rg.loss - ro["loss"]) <= 1e-5 * max(1.0, abs(ro["loss"]))
    g, go = rg.grads.astype(np.float64), ro["grads"]
    assert np.all(np.abs(g - go) <= 1e-5 * np.maximum(1.0, np.abs(go))), (env_paths, np.abs(g - go).max())
    assert np.linalg.norm(g - go) <= 1e-5 * np.linalg.norm(go) + 1e-7, (env_paths, np.linalg.norm(g - go))


@pytest.mark.parametrize("env_paths", ["pair+fused"], indirect=True)
@pytest.mark.parametrize("h0_scale", [40.0, 1e-3])
def test_loss_gradient_parity_fp16x2_h0_range(env_paths, h0_scale):
    """The fp16x2 forward step GEMM scales h by 2^(14 - floor(log2 max(1, max|h0|)))
    (stepgemm.cu hscale_kernel): an initial state far outside the tanh range (|h0| up
    to ~100) must not overflow fp16, and a tiny one must stay exact.  At x40 the fp32
    path itself sits above the 1e-5 bar against the double oracle (gradients ~40x
    larger), so there the fp16x2 error must not exceed the 3xTF32 error
    (VER_TC_F16=0) by more than 25%; at 1e-3 the usual bar holds."""
    import os
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from test_gpu_parity import _model
    H = 512
    cfg = _model(H, H)
    p = O.params_init(cfg, O.mix(3, 0x9A9A)).astype(np.float32).astype(np.float64)
    vg, vo, _ = close_both(16, 24, H, seed=33)
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    hv = vo.to_host()
    bo = O.pack(hv.seqs)
    bg = V.pack(vg, V.SequenceGroup(hv.seqs))
    h0 = (np.stack([hv.h0[s[4]] for s in bo.seqs]) * h0_scale).astype(np.float32).astype(np.float64)
    ro = O.ppo_loss(cfg, p, vo, bo, V.PPOConfig(), 0.01, h0, True)
    go = ro["grads"]
    errs = {}
    for f16 in ("1", "0"):
        os.environ["VER_TC_F16"] = f16
        try:
            rg = V.ppo_loss(cfg, p, vg, bg, V.PPOConfig(), 0.01, h0, True)
        finally:
            os.environ.pop("VER_TC_F16", None)
        assert np.isfinite(rg.loss) and np.all(np.isfinite(rg.grads))
        errs[f16] = (abs(rg.loss - ro["loss"]), np.abs(rg.grads.astype(np.float64) - go).max())
    if h0_scale < 1:
        assert errs["1"][0] <= 1e-5 * max(1.0, abs(ro["loss"]))
        assert errs["1"][1] <= 1e-5 * max(1.0, np.abs(go).max()), errs
    else:
        assert errs["1"][0] <= 1.25 * errs["0"][0] + 1e-7, errs
        assert errs["1"][1] <= 1.25 * errs["0"][1] + 1e-7, errs


@pytest.mark.parametrize("EH", [(160, 160), (96, 224)])
def test_loss_gradient_parity_fp16x2_odd_widths(EH):
    """fp16x2 GEMMs with K and N that are not multiples of the 64-element stage or
    the 256-column pair tile (zero-filled TMA boxes, masked epilogue columns): loss and
    gradients of one packed minibatch (S = 384 rows) against the oracle."""
    import paper_2210_05064_b200 as V
    from oracle import oracle as O
    from test_gpu_parity import _model
    E, H = EH
    cfg = _model(E, H)
    p = O.params_init(cfg, O.mix(5, 0x9A9A)).astype(np.float32).astype(np.float64)
    vg, vo, _ = close_both(16, 24, H, seed=35)
    V.compute_gae(vg, 0.99, 0.95)
    O.compute_gae(vo, 0.99, 0.95)
    hv = vo.to_host()
    bo = O.pack(hv.seqs)
    bg = V.pack(vg, V.SequenceGroup(hv.seqs))
    h0 = np.stack([hv.h0[s[4]] for s in bo.seqs])
    ro = O.ppo_loss(cfg, p, vo, bo, V.PPOConfig(), 0.01, h0, True)
    rg = V.ppo_loss(cfg, p, vg, bg, V.PPOConfig(), 0.01, h0, True)
    assert abs(rg.loss - ro["loss"]) <= 1e-5 * max(1.0, abs(ro["loss"]))
    g, go = rg.grads.astype(np.float64), ro["grads"]
    assert np.all(np.abs(g - go) <= 1e-5 * np.maximum(1.0, np.abs(go))), np.abs(g - go).max()
