"""GPU parity on the boundaries of the method's parameter space (readings R3-R5,
R13, R14): the widest lattice window the ABI allows (n + m_n^+ = 63 bits, M_n = 32), a complete
codebook (q = 2^n), no deletions (Pd = 0: the non-rescaled lattice), a maximally noisy
substitution channel, single-symbol frames, and an empty batch -- each in all three storage
schedules against the FP64 oracle at the north-star tolerance."""
import numpy as np
import pytest
import torch

import bsidgen
from .test_gpu_parity import assert_parity, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

EDGES = {
    # n = 32, corridor [0, 31]: 32 diagonals, window n + m_n^+ = 63 bits (kMaxWindow 64, kMaxMn 32)
    "max_window": dict(q=3, n=32, N=3, Pi=0.02, Pd=0.02, Ps=0.01, mn=(0, 31), mt=(-3, 40)),
    # every n-bit word is a codeword (q = 2^n)
    "full_codebook": dict(q=16, n=4, N=20, Pi=0.05, Pd=0.05, Ps=0.02),
    # no deletions: Pd = 0 (the G = F / Pd^r rescaling is not available, generic core)
    "no_deletions": dict(q=8, n=6, N=15, Pi=0.03, Pd=0.0, Ps=0.01),
    # substitutions only at Ps = 0.5: the received bits carry no information, L = priors
    "uninformative": dict(q=8, n=5, N=10, Pi=0.0, Pd=0.0, Ps=0.5),
    # one symbol per frame (N = 1): L_0(D) = P(D) R(Y | C_0(D)) / sum
    "single_symbol": dict(q=32, n=8, N=1, Pi=0.05, Pd=0.05, Ps=0.0),
}


@pytest.mark.parametrize("name", sorted(EDGES))
def test_edge_configuration(name):
    kw = dict(EDGES[name])
    cfg = bsidgen.Config(name, frames=0, seed=777, priors=(name == "single_symbol"), **kw)
    b = bsidgen.make_batch(cfg, 0, 7)
    res = run_oracle(cfg, b)
    for mode in (1, 2, 3):
        _, L, st = run_gpu(cfg, b, mode)
        assert_parity(L, st, res)
    if name == "uninformative":  # Ps = 1/2 and no insertions/deletions: the APPs are the (uniform) priors
        _, L, _ = run_gpu(cfg, b, 3)
        np.testing.assert_allclose(L, 1.0 / cfg.q, rtol=1e-5)


def test_empty_batch():
    from paper_1802_08483_b200 import Decoder
    cfg = bsidgen.configs()["C1"]
    d = Decoder.from_config(cfg, bsidgen.codebook(cfg), device=0)
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    L, st = d.decode(torch.zeros(1, dtype=torch.int32, device="cuda"), torch.empty(0, dtype=torch.int64, device="cuda"), e)
    torch.cuda.synchronize()
    assert L.shape == (0, cfg.N, cfg.q) and st.shape == (0,)
    assert d.last_launch_count() == 0


def test_c_example_runs():
    """examples/decode_host (plain C, host buffers through bsidmap_decode_batch_host) decodes its
    256 C1-shaped frames with every frame OK and a small symbol error rate."""
    import os
    import re
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["make", "-C", root, "examples/decode_host"], check=True, capture_output=True)
    r = subprocess.run([os.path.join(root, "examples", "decode_host")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    ser = float(re.search(r"symbol error rate ([0-9.]+)", r.stdout).group(1))
    assert ser < 0.05, r.stdout


@pytest.mark.parametrize("shape,seed", [(s, k) for s in ("C1", "C2", "C3", "C4", "C5") for k in range(2)])
def test_spec_shapes_random_channels(shape, seed):
    """Each specialised lattice shape (n, m_n^-, M_n) of C1-C5 with a random channel around its
    own (Pi, Pd, Ps > 0 for every shape), random priors on or off and a short frame, in the
    three storage schedules and the auto plan, against the oracle."""
    rng = np.random.default_rng(100 + seed)
    base = bsidgen.configs()[shape]
    Pi = float(base.Pi * rng.uniform(0.5, 1.5))
    Pd = float(base.Pd * rng.uniform(0.5, 1.5))
    Ps = float(rng.choice([0.0, 0.003, 0.02]))
    N = int(rng.integers(3, 9))
    cfg = bsidgen.Config(f"{shape}r{seed}", q=base.q, n=base.n, N=N, Pi=Pi, Pd=Pd, Ps=Ps, frames=0,
                         priors=bool(rng.random() < 0.5), mn=base.mn,
                         mt=(min(base.mn[0], -3 * base.n), max(base.mn[1], 3 * base.n)), seed=500 + seed)
    b = bsidgen.make_batch(cfg, 0, int(rng.integers(2, 7)))
    res = run_oracle(cfg, b)
    for mode in (0, 1, 2, 3):
        d, L, st = run_gpu(cfg, b, mode)
        assert d.plan(len(b.rho))["core"] == "spec"
        assert_parity(L, st, res)


def test_large_alphabet_uses_generic_core(monkeypatch):
    monkeypatch.setenv("BSIDMAP_JIT", "0")
    """q = 512 on C2's lattice shape: the specialised APP kernels would need more shared memory than
    a CTA has, so the decoder takes the generic core; parity against the oracle in all schedules."""
    cfg = bsidgen.Config("bigq", q=512, n=10, N=3, Pi=0.01, Pd=0.01, Ps=0.001, frames=0, seed=31,
                         mn=(-6, 7), mt=(-12, 12))
    b = bsidgen.make_batch(cfg, 0, 3)
    res = run_oracle(cfg, b)
    for mode in (0, 1, 2, 3):
        d, L, st = run_gpu(cfg, b, mode)
        assert d.plan(3)["core"] == "generic"
        assert_parity(L, st, res)


@pytest.mark.parametrize("shape,q", [("C5", 25), ("C2", 7), ("C3", 31)])
def test_odd_alphabet_local_schedule(shape, q):
    """Odd q on a specialised shape with M_tau <= 64 (the warp-per-frame local schedule): the per-warp
    shared-memory slices must keep the FP64 rows 8-byte aligned (found by tools/stress.py)."""
    base = bsidgen.configs()[shape]
    cfg = bsidgen.Config(f"odd{shape}", q=q, n=base.n, N=5, Pi=0.02, Pd=0.02, Ps=0.01, frames=0, seed=63,
                         mn=base.mn, mt=(base.mn[0] - 6, base.mn[1] + 7))
    b = bsidgen.make_batch(cfg, 0, 24)
    res = run_oracle(cfg, b)
    for mode in (2, 3):
        d, L, st = run_gpu(cfg, b, mode)
        assert_parity(L, st, res)
    assert d.plan(24)["core"] == "spec"


def test_chunked_overlapped_c5_shape_bit_identical():
    """C5's shape (scalar core, CTA alpha/beta, priors) decoded in one call and in chunks of two frames
    (each chunk's alpha/beta on the side stream, two sub-batches of one frame): identical L."""
    full = bsidgen.configs()["C5"]
    cfg = bsidgen.Config("C5c", q=full.q, n=full.n, N=150, Pi=full.Pi, Pd=full.Pd, Ps=full.Ps, frames=0,
                         priors=True, mn=full.mn, mt=full.mt, seed=full.seed)
    b = bsidgen.make_batch(cfg, 0, 6)
    d1, L1, st1 = run_gpu(cfg, b, 0)
    assert d1.plan(6)["alpha_beta_overlap_subbatches"] == 2
    per = d1.workspace_bytes(1, 0)
    d2, L2, st2 = run_gpu(cfg, b, 0, ws_limit=2 * per + 1024)
    assert d2.plan(6)["chunks"] == 3
    np.testing.assert_array_equal(st2, st1)
    np.testing.assert_array_equal(L2, L1)
    assert (st1 == 0).all()


def test_cta_alpha_beta_ring_depth_bit_identical():
    """C4's shape (M_tau = 611: the CTA alpha/beta kernel, ~M_tau/2 threads): 640 frames in one call
    (grid of 1280 CTAs >= 4 per SM: single-stage Gamma ring) and in chunks of 64 frames (deep ring)
    give identical L; the first frames match the oracle."""
    full = bsidgen.configs()["C4"]
    cfg = bsidgen.Config("C4r", q=full.q, n=full.n, N=12, Pi=full.Pi, Pd=full.Pd, Ps=full.Ps, frames=0,
                         mn=full.mn, mt=full.mt, seed=full.seed)
    F = 640
    b = bsidgen.make_batch(cfg, 0, F)
    d1, L1, st1 = run_gpu(cfg, b, 0)
    plan = d1.plan(F)
    assert plan["chunks"] == 1 and plan["alpha_beta_block"] == 320
    per = d1.workspace_bytes(1, 0)
    d2, L2, st2 = run_gpu(cfg, b, 0, ws_limit=64 * per + 1024)
    assert d2.plan(F)["chunks"] == 10
    np.testing.assert_array_equal(st2, st1)
    np.testing.assert_array_equal(L2, L1)
    assert_parity(L1, st1, run_oracle(cfg, b, frames=[0, 1]), frames=[0, 1])


def _floor_priors(b, rng):
    """Priors spanning ~30 decades: the transmitted symbol 1, every other symbol 10^-u with u drawn
    in [12, 27] -- the oracle's L then has many entries between ~1e-35 and ~1e-20, around the 1e-30
    floor of the relative-error gate (reading R11)."""
    F, N = b.msg.shape
    q = b.cfg.q
    u = rng.uniform(12.0, 27.0, size=(F, N, q))
    P = 10.0 ** -u
    np.put_along_axis(P, b.msg[:, :, None].astype(np.int64), 1.0, axis=2)
    P /= P.sum(2, keepdims=True)
    return P.astype(np.float32)


@pytest.mark.parametrize("name,N,frames", [("C2", 100, 6), ("C1", 10, 40), ("C5", 24, 2)])
def test_app_dynamic_range_near_the_floor(name, N, frames):
    """L entries near the 1e-30 floor (R11), fed by extreme priors and by low-weight windows
    (windows far from the posterior drift carry alpha*beta weights many decades below the tile's
    largest): the per-window FP32 terms, the FP64 sums over windows and symbols and the FP64
    normalisation must hold the 1e-4 relative gate there too.  Both spec APP cores: the pair core
    (C1, C2 shapes) and the scalar core (C5 shape, several rounds of live windows per frame)."""
    import dataclasses
    cfg = dataclasses.replace(bsidgen.configs()[name], N=N, priors=True)
    b = bsidgen.make_batch(cfg, 5, frames)
    b.priors = _floor_priors(b, np.random.default_rng(11))
    res = run_oracle(cfg, b)
    Lo = np.concatenate([r["L"].ravel() for r in res])
    near = ((Lo > 1e-34) & (Lo < 1e-26)).sum()
    assert near >= 20, near   # the case really exercises the floor
    for mode in (2, 3):
        _, L, st = run_gpu(cfg, b, mode)
        assert_parity(L, st, res)


def test_wide_trellis_alpha_beta_reads_gamma_from_global():
    """A trellis whose Gamma_i block (M_n x M_tau FP32) exceeds shared memory -- C4's code and
    channel (M_n = 26) with M_tau = 2401 (the width C4's channel needs at N ~ 1.5e5): the CTA alpha/beta
    recursion reads Gamma_i from global memory instead of the TMA ring (every schedule
    used to fail with EPLAN there).  Against the FP64 oracle in the Gamma-sum and stored schedules."""
    import dataclasses
    cfg = dataclasses.replace(bsidgen.configs()["C4"], N=12, mt=(-1200, 1200))
    assert cfg.Mn * ((cfg.Mt + 7) // 8 * 8) * 4 > 227 * 1024
    b = bsidgen.make_batch(cfg, 3, 3)
    res = run_oracle(cfg, b)
    for mode in (3, 1):
        d, L, st = run_gpu(cfg, b, mode)
        assert_parity(L, st, res)
