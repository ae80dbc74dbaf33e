"""tcgen05 GEMM (TMA + TMEM, 3xTF32 / 1xTF32) vs float64 numpy, all operand
majors and split-K; the SIMT fp32 GEMM as a second reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128, 32), (256, 384, 512), (16384, 512, 512), (300, 200, 100), (512, 1536, 4096),
          (1, 512, 512), (7, 1536, 512), (50, 512, 1536), (33, 20, 12)]


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_tc_gemm_3xtf32(ta, tb, M, N, K):
    import paper_2210_05064_b200 as V
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    ref = (A.astype(np.float64).T if ta else A.astype(np.float64)) @ (B.astype(np.float64).T if tb else B)
    scale = np.sqrt(K)  # |C| ~ sqrt(K): errors below are relative to the output scale
    C0 = V.debug_gemm(A, B, ta, tb, engine=0)
    err0 = np.abs(C0 - ref).max() / scale  # fp32 SIMT
    assert err0 < 3e-5
    for split in (1, 4):
        C3 = V.debug_gemm(A, B, ta, tb, engine=1, splitk=split)
        err3 = np.abs(C3 - ref).max() / scale
        # fp32-grade: hi = trunc_tf32(x) (the tensor core's own read of fp32), lo = x - hi;
        # the dropped lo*lo term is <= 2^-20 |ab| per product
        assert err3 < max(1e-5, 3 * err0), (split, err3, err0)
    C1 = V.debug_gemm(A, B, ta, tb, engine=2)
    err1 = np.abs(C1 - ref).max() / scale
    assert err1 < 1e-2, err1  # tf32 (10-bit mantissa) inputs


def test_presplit_weight_operand_bit_identical(monkeypatch):
    """The weights' lo operand loaded pre-split by TMA (VER_TC_BLO=1, default: the
    encoder / projection GEMMs and the recurrence step kernel's U) gives the same
    bits as splitting B in shared memory (VER_TC_BLO=0): one full update."""
    import paper_2210_05064_b200 as V
    from paper_2210_05064_b200 import synth
    from paper_2210_05064_b200.rng import mix
    T, N, E, H = 32, 24, 256, 256
    cfg = V.ModelConfig(obs_dim=2, encoder_dim=E, hidden_dim=H, action_kind=0, num_actions=2)
    p = V.params_init(cfg, mix(2, 0x9A9A)).astype(np.float32)
    wl = synth.make_workload(T, N, obs_dim=2, num_actions=2, hidden_dim=H, seed=3)
    # big recurrence steps from 6 rows: the persistent step kernel's U operand too
    monkeypatch.setenv("VER_REC_BIG_FWD", "6")
    monkeypatch.setenv("VER_REC_BIG_BWD", "6")
    out = []
    for blo in ("1", "0"):
        monkeypatch.setenv("VER_TC_BLO", blo)
        lg = V.Learner(cfg, p, V.PPOConfig(epochs=2, minibatches=2), run_seed=mix(2, 0xF00D))
        buf = V.RolloutBuffer(T, N, V.VARIABLE, 0, 2, 0, H)
        synth.fill_buffer(buf, wl)
        lg.update(buf.close_rollout())
        out.append(lg.params())
    np.testing.assert_array_equal(out[0], out[1])


@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("M,N,K", [(512, 1536, 4096), (300, 200, 100), (33, 20, 12)])
def test_mn_major_a_via_tmem_bit_identical(monkeypatch, tb, M, N, K):
    """MN-major A moved into tensor memory by the split warps (VER_TC_ATM_MN=1,
    default: the weight-gradient GEMMs) gives the same bits as A read from the
    swizzled shared-memory tile (VER_TC_ATM_MN=0): same hi / lo operands, same
    MMA order."""
    import paper_2210_05064_b200 as V
    rng = np.random.default_rng(M + 3 * N + 7 * K)
    A = rng.standard_normal((K, M)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    out = []
    for on in ("1", "0"):
        monkeypatch.setenv("VER_TC_ATM_MN", on)
        out.append([V.debug_gemm(A, B, True, tb, engine=1, splitk=s) for s in (1, 4)])
    for a, b in zip(*out):
        np.testing.assert_array_equal(a, b)
