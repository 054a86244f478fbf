"""GPU parity of the SURVEY 8(f) NEXT rows built on the decoder:
NEXT-1 soft frame-boundary priors (alpha_0, beta_N as distributions, Phi_T on device),
NEXT-4 extrinsic output; against the FP64 oracle (pinned in test_oracle_pins.py)."""
import numpy as np
import pytest
import torch

import bsidgen
import oracle
from tests.test_gpu_parity import FLOOR, TOL, _dec, run_oracle, small_cfg, to_dev

pytestmark = pytest.mark.gpu


def _cfg(name, **kw):
    """C1/C2 as configured; "C3r", "C4r", "C5r": that config's code, channel, corridor and trellis
    (M_tau 267 / 611 / 906: CTA alpha/beta, scalar or register-heavy APP kernels, the CTA local
    schedule) with N cut to 24 so the oracle stays fast."""
    if name.endswith("r"):
        full = bsidgen.configs()[name[:-1]]
        return small_cfg(name[:-1], N=24, mn=full.mn, mt=full.mt, **kw)
    return small_cfg(name, **kw)


def _soft_batch(cfg, F, seed):
    """Frames whose received sequence carries extra random bits before and after the
    frame, decoded with a start-drift prior and end-drift weights over the states."""
    rng = np.random.default_rng(seed)
    b = bsidgen.make_batch(cfg, 100 + seed, F)
    wpf = b.rx.shape[1] + 2
    rx = np.zeros((F, wpf), np.uint32)
    rho = np.zeros(F, np.int32)
    bits_all = []
    for f in range(F):
        pre = rng.integers(0, 2, int(rng.integers(0, 3)))
        post = rng.integers(0, 2, int(rng.integers(0, 3)))
        bits = np.concatenate([pre, b.bits(f), post]).astype(np.uint8)
        bits_all.append(bits)
        rx[f] = bsidgen.pack_bits(bits, wpf)
        rho[f] = len(bits)
    b.rx, b.rho, b.offsets = rx, rho, np.arange(F, dtype=np.int64) * wpf
    Mt = cfg.Mt
    a0 = np.zeros((F, Mt))
    a0[:, -cfg.mt[0]:-cfg.mt[0] + 3] = rng.random((F, 3)) + 0.1  # start drift 0, 1 or 2
    bN = rng.random((F, Mt)) + 1e-3
    return b, a0, bN


@pytest.mark.parametrize("name,mode", [("C1", 1), ("C1", 2), ("C1", 3), ("C2", 2), ("C2", 3), ("C3r", 0),
                                       ("C3r", 2), ("C4r", 0), ("C4r", 2), ("C5r", 0), ("C5r", 2)])
def test_soft_boundary_priors_parity(name, mode):
    cfg = _cfg(name)
    b, a0, bN = _soft_batch(cfg, 12, seed=hash(name) % 97)
    d = _dec().from_config(cfg, b.C, mode=mode, device=0)
    rx, off, rho, pri = to_dev(b)
    dev = torch.device("cuda", 0)
    L, st = d.decode(rx, off, rho, pri, alpha0=torch.from_numpy(a0).to(dev), betaN=torch.from_numpy(bN).to(dev))
    L, st = L.cpu().numpy().astype(np.float64), st.cpu().numpy()
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    worst = 0.0
    for f in range(12):
        pf = b.priors[f].astype(np.float64) if b.priors is not None else None
        r = oracle.decode(prob, b.bits(f), pf, alpha0=a0[f], betaN=bN[f])
        assert st[f] == r["status"]
        if r["status"] != oracle.OK:
            continue
        worst = max(worst, float((np.abs(L[f] - r["L"]) / np.maximum(r["L"], FLOOR)).max()))
    assert worst <= TOL, worst


def test_soft_boundary_generic_core(monkeypatch):
    monkeypatch.setenv("BSIDMAP_JIT", "0")
    cfg = bsidgen.Config("S", q=5, n=4, N=9, Pi=0.03, Pd=0.02, Ps=0.01, frames=0, seed=77)
    b, a0, bN = _soft_batch(cfg, 9, seed=5)
    d = _dec().from_config(cfg, b.C, mode=3, device=0)
    assert d.plan(9)["core"] == "generic"
    rx, off, rho, pri = to_dev(b)
    dev = torch.device("cuda", 0)
    L, st = d.decode(rx, off, rho, pri, alpha0=torch.from_numpy(a0).to(dev), betaN=torch.from_numpy(bN).to(dev))
    L, st = L.cpu().numpy().astype(np.float64), st.cpu().numpy()
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    for f in range(9):
        r = oracle.decode(prob, b.bits(f), alpha0=a0[f], betaN=bN[f])
        assert st[f] == r["status"]
        if r["status"] == oracle.OK:
            assert (np.abs(L[f] - r["L"]) / np.maximum(r["L"], FLOOR)).max() <= TOL


@pytest.mark.parametrize("name,mode", [("C1", 3), ("C2", 2), ("C2", 3), ("C3r", 0), ("C4r", 0), ("C5r", 0),
                                       ("C5r", 2)])
def test_extrinsic_parity(name, mode):
    cfg = _cfg(name, priors=True)
    b = bsidgen.make_batch(cfg, 0, 10)
    b.priors[1, 2, :] = 0.0
    b.priors[1, 2, 0] = 1.0
    b.priors[3, 4, 1] = 0.0
    d = _dec().from_config(cfg, b.C, mode=mode, device=0)
    rx, off, rho, pri = to_dev(b)
    L, st, E = d.decode(rx, off, rho, pri, extrinsic=True)
    E = E.cpu().numpy().astype(np.float64)
    res = run_oracle(cfg, b)
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    for f in range(10):
        r = oracle.decode(prob, b.bits(f), b.priors[f].astype(np.float64), extrinsic=True)
        err = np.abs(E[f] - r["E"]) / np.maximum(r["E"], FLOOR)
        assert err.max() <= TOL, (f, err.max())
    assert E[3, 4, 1] == 0.0
    np.testing.assert_allclose(E.sum(2), 1.0, atol=1e-5)


def test_phi_on_device_equals_host_pmf():
    from paper_1802_08483_b200 import drift_pmf, phi
    for T, Pi, Pd, lo, hi in [(70, 0.01, 0.01, -11, 11), (1000, 0.01, 0.01, -31, 31), (120000, 0.02, 0.02, -452, 453)]:
        dev = phi(T, Pi, Pd, lo, hi, 3, device=0).cpu().numpy()
        host = drift_pmf(T, Pi, Pd, lo, hi)
        for f in range(3):
            np.testing.assert_array_equal(dev[f], host)
        assert host.sum() > 1 - 1e-9
