"""The slab schedule (RECOMPUTE on the spec cores, reading R19): Gamma kept for two
slabs of symbol indices, alpha through each slab of a forward sweep, Gamma recomputed only where
alpha_i(m') != 0 in a backward sweep that runs beta and the live-window APP.  Against the FP64 oracle
at the north-star gate over slab lengths (one index per slab to the whole frame, ragged last slabs),
with and without the alpha-support skip, chunked, with soft frame boundaries, and with a frame that
becomes impossible in the middle of the forward sweep."""
import numpy as np
import pytest
import torch

import bsidgen
import oracle
from tests.test_gpu_parity import assert_parity, run_gpu, run_oracle, small_cfg, to_dev, _dec, FLOOR, TOL

pytestmark = pytest.mark.gpu


def _slab(monkeypatch, cfg, b, length, askip=True, ws_limit=None):
    monkeypatch.setenv("BSIDMAP_SLAB_LEN", str(length))
    monkeypatch.setenv("BSIDMAP_SLAB_ASKIP", "1" if askip else "0")
    d, L, st = run_gpu(cfg, b, 2, ws_limit=ws_limit)
    plan = d.plan(len(b.rho))
    assert plan["mode"] == "recompute-slab" and plan["slab"] == min(length, cfg.N)
    return d, L, st


@pytest.mark.parametrize("name,frames,lengths", [("C1", 40, [1, 3, 10]), ("C2", 24, [7, 8, 100]),
                                                 ("C3", 3, [5, 16]), ("C5r", 2, [8, 13])])
def test_slab_lengths_parity(name, frames, lengths, monkeypatch):
    if name == "C5r":
        full = bsidgen.configs()["C5"]
        cfg = small_cfg("C5", N=40, mn=full.mn, mt=full.mt)
    else:
        cfg = small_cfg(name)
    b = bsidgen.make_batch(cfg, 21, frames)
    res = run_oracle(cfg, b)
    _, Lg, stg = run_gpu(cfg, b, 3)
    for length in lengths:
        for askip in (True, False):
            _, L, st = _slab(monkeypatch, cfg, b, length, askip)
            assert_parity(L, st, res)
            np.testing.assert_array_equal(st, stg)
            np.testing.assert_allclose(L, Lg, rtol=2e-5, atol=1e-30)


def test_slab_chunked_bit_identical(monkeypatch):
    """Chunking the batch does not change the arithmetic at a fixed slab length (and a fixed number
    of frames per APP warp, whose FP64 association otherwise follows the launch size) when every
    window is recomputed; with the alpha-support skip the skipped warps follow the packing of frames
    into warps, which changes beta only where alpha = 0 (R19): L equal up to rounding."""
    monkeypatch.setenv("BSIDMAP_APP_G", "1")
    cfg = small_cfg("C4")
    b = bsidgen.make_batch(cfg, 4, 6)
    for askip in (False, True):
        d, L1, st1 = _slab(monkeypatch, cfg, b, 16, askip)
        per = d.workspace_bytes(1, 2)
        d2, L2, st2 = _slab(monkeypatch, cfg, b, 16, askip, ws_limit=per * 2 + per // 2)
        assert d2.plan(6)["chunks"] == 3
        np.testing.assert_array_equal(st1, st2)
        if askip:
            np.testing.assert_allclose(L1, L2, rtol=2e-5, atol=1e-30)
        else:
            np.testing.assert_array_equal(L1, L2)
    assert_parity(L1, st1, run_oracle(cfg, b, [0, 5]), [0, 5])


def test_slab_soft_boundaries(monkeypatch):
    """Start-drift prior alpha_0 and end weights beta_N (NEXT-1) through a multi-slab decode."""
    from tests.test_gpu_next import _cfg, _soft_batch
    cfg = _cfg("C4r")
    b, a0, bN = _soft_batch(cfg, 6, seed=5)
    monkeypatch.setenv("BSIDMAP_SLAB_LEN", "5")
    d = _dec().from_config(cfg, b.C, mode=2, device=0)
    assert d.plan(6)["slab"] == 5
    rx, off, rho, pri = to_dev(b)
    dev = torch.device("cuda", 0)
    L, st = d.decode(rx, off, rho, pri, alpha0=torch.from_numpy(a0).to(dev), betaN=torch.from_numpy(bN).to(dev))
    L, st = L.cpu().numpy().astype(np.float64), st.cpu().numpy()
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    res = [oracle.decode(prob, b.bits(f), None, alpha0=a0[f], betaN=bN[f]) for f in range(6)]
    assert_parity(L, st, res)


def test_slab_underflow_mid_frame(monkeypatch):
    """No drift allowed (m_n = m_tau = [0, 0]) and no substitutions: frame 2's symbol 5 matches no
    codeword, so alpha underflows in the second slab of the forward sweep; the frame is reported
    UNDERFLOW with a zero L and the other frames decode their transmitted symbols with probability 1.
    (Pd > 0: the rescaled lattice of the run-time compiled core, which the slab schedule needs.)"""
    cfg = small_cfg("C1", Pi=0.001, Pd=0.001, Ps=0.0, mn=(0, 0), mt=(0, 0))
    b = bsidgen.make_batch(cfg, 0, 4)
    C5 = set(int(w) for w in b.C[5])
    bad = next(w for w in range(1 << cfg.n) if w not in C5)
    bits = b.bits(2)
    bits[5 * cfg.n:6 * cfg.n] = [(bad >> t) & 1 for t in range(cfg.n)]
    b.rx[2] = bsidgen.pack_bits(bits, b.rx.shape[1])
    res = run_oracle(cfg, b)
    assert res[2]["status"] == oracle.UNDERFLOW
    _, L, st = _slab(monkeypatch, cfg, b, 3)
    assert_parity(L, st, res)
    for f in (0, 1, 3):
        np.testing.assert_allclose(L[f][np.arange(cfg.N), b.msg[f]], 1.0, rtol=0, atol=1e-6)
