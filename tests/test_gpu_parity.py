"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on the
same seeded inputs.  Gate (north star / DESIGN.md reading R11):
  err = |L_gpu - L_orc| / max(L_orc, 1e-30) <= 1e-4 on every entry,
  hard decisions equal wherever the oracle's top-two gap exceeds 1e-3,
  frame status equal.
"""
import os

import numpy as np
import pytest
import torch

import bsidgen
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-4
FLOOR = 1e-30


def _dec():
    from paper_1802_08483_b200 import Decoder
    return Decoder


def to_dev(b):
    dev = torch.device("cuda", 0)
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    return rx, off, rho, pri


def run_gpu(cfg, b, mode=0, ws_limit=None):
    Decoder = _dec()
    d = Decoder.from_config(cfg, b.C, mode=mode, device=0)
    if ws_limit:
        d.set_workspace_limit(ws_limit)
    rx, off, rho, pri = to_dev(b)
    L, st = d.decode(rx, off, rho, pri)
    torch.cuda.synchronize()
    return d, L.cpu().numpy().astype(np.float64), st.cpu().numpy()


def run_oracle(cfg, b, frames=None):
    frames = range(len(b.rho)) if frames is None else frames
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    ys = [b.bits(f) for f in frames]
    pl = [b.priors[f].astype(np.float64) if b.priors is not None else None for f in frames]
    return oracle.decode_many(prob, ys, pl)


def assert_parity(L_gpu, st_gpu, res, frames=None):
    frames = range(len(res)) if frames is None else frames
    worst = 0.0
    for k, f in enumerate(frames):
        r = res[k]
        assert st_gpu[f] == r["status"], (f, st_gpu[f], r["status"])
        if r["status"] != oracle.OK:
            assert not L_gpu[f].any()
            continue
        Lo, Lg = r["L"], L_gpu[f]
        err = np.abs(Lg - Lo) / np.maximum(Lo, FLOOR)
        worst = max(worst, float(err.max()))
        srt = np.sort(Lo, axis=1)
        decided = (srt[:, -1] - srt[:, -2]) > 1e-3
        np.testing.assert_array_equal(np.argmax(Lg, 1)[decided], np.argmax(Lo, 1)[decided])
    assert worst <= TOL, f"max relative error {worst:.3e} > {TOL}"
    return worst


def small_cfg(name, **kw):
    cfg = bsidgen.configs()[name]
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


# ------------------------------------------------------------------ configs

@pytest.mark.parametrize("mode", [1, 2, 3])
def test_c1_parity(mode):
    cfg = small_cfg("C1")
    b = bsidgen.make_batch(cfg, 0, 300)     # 300 x 23 lanes: many tiles + ragged tail
    d, L, st = run_gpu(cfg, b, mode)
    assert d.plan(300)["core"] == "spec"
    assert_parity(L, st, run_oracle(cfg, b))


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_c2_parity(mode):
    cfg = small_cfg("C2")
    b = bsidgen.make_batch(cfg, 1000, 48)
    d, L, st = run_gpu(cfg, b, mode)
    assert d.plan(48)["core"] == "spec"
    assert_parity(L, st, run_oracle(cfg, b))


# RECOMPUTE's two schedules: the slab schedule (spec cores; slabs of 8 symbol indices here, so the
# frames span many slabs and a ragged last one) and the paper's per-frame local kernels
SCHEDS = {"slab": ({"BSIDMAP_SLAB_LEN": "8"}, "recompute-slab"),
          "local": ({"BSIDMAP_SLAB": "0"}, "recompute-local")}


def run_recompute(cfg, b, sched, monkeypatch):
    env, mode_name = SCHEDS[sched]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    d, L, st = run_gpu(cfg, b, 2)
    assert d.plan(len(b.rho))["mode"].startswith(mode_name)
    if sched == "slab":
        assert d.plan(len(b.rho))["slab"] == min(8, cfg.N)
    for k in env:
        monkeypatch.delenv(k)
    return d, L, st


@pytest.mark.parametrize("sched", ["slab", "local"])
def test_c3_parity(sched, monkeypatch):
    cfg = small_cfg("C3")
    b = bsidgen.make_batch(cfg, 7, 4)
    _, L, st = run_recompute(cfg, b, sched, monkeypatch)
    assert_parity(L, st, run_oracle(cfg, b))


@pytest.mark.parametrize("sched", ["slab", "local"])
def test_c4_parity(sched, monkeypatch):
    cfg = small_cfg("C4")
    b = bsidgen.make_batch(cfg, 3, 2)
    _, L, st = run_recompute(cfg, b, sched, monkeypatch)
    assert_parity(L, st, run_oracle(cfg, b))


@pytest.mark.parametrize("sched", ["slab", "local"])
def test_c5_shape_parity_reduced_N(sched, monkeypatch):
    """C5's q, n, channel, corridor, M_tau and non-uniform priors, N cut to 60 so the
    oracle finishes in seconds (full-N C5 is checked by sampled gamma + properties)."""
    full = bsidgen.configs()["C5"]
    cfg = small_cfg("C5", N=60, mn=full.mn, mt=full.mt)
    b = bsidgen.make_batch(cfg, 0, 2)
    _, L, st = run_recompute(cfg, b, sched, monkeypatch)
    assert_parity(L, st, run_oracle(cfg, b))


@pytest.mark.parametrize("sched", ["slab", "local"])
def test_c2_recompute_parity(sched, monkeypatch):
    cfg = small_cfg("C2")
    b = bsidgen.make_batch(cfg, 1000, 48)   # N = 100: twelve slabs of 8 and a ragged one of 4
    _, L, st = run_recompute(cfg, b, sched, monkeypatch)
    assert_parity(L, st, run_oracle(cfg, b))


# ------------------------------------------------------- element-wise gamma

@pytest.mark.parametrize("name,frames,idx", [("C1", 5, [0, 4, 9]), ("C2", 3, [0, 37, 99]),
                                              ("C4", 1, [0, 500, 999]), ("C5", 1, [0, 5000, 9999])])
def test_gamma_elementwise(name, frames, idx):
    cfg = small_cfg(name)
    b = bsidgen.make_batch(cfg, 11, frames)
    d = _dec().from_config(cfg, b.C, device=0)
    rx, off, rho, pri = to_dev(b)
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    for i in idx:
        g = d.debug_gamma(rx, off, rho, pri, i).cpu().numpy()
        for f in range(frames):
            go = oracle.gamma(prob, b.bits(f), i, b.priors[f] if b.priors is not None else None)
            zero = go == 0
            assert not g[f][zero].any(), "structural zeros must match exactly"
            err = np.abs(g[f] - go) / np.maximum(go, FLOOR)
            assert err.max() <= 1e-5, (i, f, err.max())


# ------------------------------------------------------------ generic core

def _random_cfg(rng, k):
    n = int(rng.integers(1, 14))
    q = int(rng.integers(2, min(40, 2 ** n) + 1))
    N = int(rng.integers(1, 30))
    p = float(rng.choice([0.0, 0.005, 0.03, 0.1]))
    Ps = float(rng.choice([0.0, 0.02]))
    cfg = bsidgen.Config(f"R{k}", q=q, n=n, N=N, Pi=p, Pd=p * float(rng.choice([0.5, 1.0, 1.5])), Ps=Ps,
                         frames=0, priors=bool(rng.random() < 0.5), seed=9000 + k)
    return cfg


@pytest.mark.parametrize("k", range(10))
def test_random_shapes_generic_core(k, monkeypatch):
    monkeypatch.setenv("BSIDMAP_JIT", "0")   # the generic core (run-time compiled cores: test_gpu_jit.py)
    rng = np.random.default_rng(k)
    cfg = _random_cfg(rng, k)
    F = int(rng.integers(1, 40))
    b = bsidgen.make_batch(cfg, 0, F)
    res = run_oracle(cfg, b)
    for mode in (1, 2, 3):
        d, L, st = run_gpu(cfg, b, mode)
        assert_parity(L, st, res)


# ------------------------------------------------------------- edge cases

def test_status_edge_cases():
    cfg = small_cfg("C1")
    b = bsidgen.make_batch(cfg, 0, 6)
    # frame 1: end drift above m_tau^+ ; frame 2: below m_tau^-
    b.rho[1] = cfg.tau + cfg.mt[1] + 1
    b.rho[2] = cfg.tau + cfg.mt[0] - 1
    b.rx = np.concatenate([b.rx, np.zeros((6, 2), np.uint32)], 1)
    b.offsets = np.arange(6, dtype=np.int64) * b.rx.shape[1]
    _, L, st = run_gpu(cfg, b, 2)
    assert st[1] == 1 and st[2] == 1
    assert_parity(L, st, run_oracle(cfg, b))


def test_underflow_status():
    """Noiseless channel with received bits matching no codeword: Y is impossible."""
    cfg = small_cfg("C1", Pi=0.0, Pd=0.0, Ps=0.0, mn=(0, 0), mt=(0, 0))
    b = bsidgen.make_batch(cfg, 0, 4)
    C0 = set(int(w) for w in b.C[0])
    bad = next(w for w in range(1 << cfg.n) if w not in C0)
    bits = b.bits(2)
    bits[:cfg.n] = [(bad >> t) & 1 for t in range(cfg.n)]
    b.rx[2] = bsidgen.pack_bits(bits, b.rx.shape[1])
    _, L, st = run_gpu(cfg, b, 2)
    res = run_oracle(cfg, b)
    assert res[2]["status"] == oracle.UNDERFLOW
    assert_parity(L, st, res)
    # noiseless: the transmitted symbols get probability 1
    for f in (0, 1, 3):
        np.testing.assert_allclose(L[f][np.arange(cfg.N), b.msg[f]], 1.0, rtol=0, atol=1e-6)


def test_binary_single_bit_codes():
    cfg = bsidgen.Config("E", q=2, n=1, N=40, Pi=0.02, Pd=0.03, Ps=0.01, frames=0, seed=5)
    b = bsidgen.make_batch(cfg, 0, 9)
    res = run_oracle(cfg, b)
    for mode in (1, 2, 3):
        _, L, st = run_gpu(cfg, b, mode)
        assert_parity(L, st, res)


def test_zero_priors_and_one_hot():
    cfg = small_cfg("C1", priors=True)
    b = bsidgen.make_batch(cfg, 0, 5)
    b.priors[:, 3, :] = 0.0
    b.priors[:, 3, 2] = 1.0
    b.priors[0, 5, :4] = 0.0
    _, L, st = run_gpu(cfg, b, 2)
    res = run_oracle(cfg, b)
    assert_parity(L, st, res)
    np.testing.assert_allclose(L[:, 3, 2], 1.0, atol=1e-6)


def test_chunked_equals_unchunked_and_host_path():
    cfg = small_cfg("C2")
    b = bsidgen.make_batch(cfg, 50, 40)
    d, L1, st1 = run_gpu(cfg, b, 3)
    per = d.workspace_bytes(1, 3)
    _, L2, st2 = run_gpu(cfg, b, 3, ws_limit=per * 7)   # 6 chunks of 7 + tail
    np.testing.assert_array_equal(st1, st2)
    np.testing.assert_allclose(L2, L1, rtol=1e-5, atol=1e-30)
    # end-to-end host path through bsidmap_decode_batch_host (pinned buffers)
    rx = torch.from_numpy(b.rx.ravel().copy()).pin_memory()
    off = torch.from_numpy(b.offsets).pin_memory()
    rho = torch.from_numpy(b.rho).pin_memory()
    L3 = torch.empty((40, cfg.N, cfg.q), dtype=torch.float32).pin_memory()
    st3 = torch.empty(40, dtype=torch.int32).pin_memory()
    d.decode_host(rx, off, rho, None, L3, st3)
    np.testing.assert_array_equal(st3.numpy(), st1)
    np.testing.assert_allclose(L3.numpy(), L1, rtol=1e-5, atol=1e-30)


@pytest.mark.parametrize("frames", [16384 + 17, 8 * 8192 + 5])
def test_host_path_subbatches(frames):
    """bsidmap_decode_batch_host splits the batch into up to 8 equal sub-batches and the last one
    again into 1/2, 1/4, 1/8, 1/8 (host path): with C1 frames (small) at 2 and 8 equal
    sub-batches plus the split tail, every frame's status equals and its L agrees (1e-5) with the
    device-buffer decode of the same frames in one call, and sampled frames match the oracle."""
    cfg = small_cfg("C1")
    b = bsidgen.make_batch(cfg, 3, frames)
    d, L1, st1 = run_gpu(cfg, b, 3)
    rx = torch.from_numpy(b.rx.ravel().copy()).pin_memory()
    off = torch.from_numpy(b.offsets).pin_memory()
    rho = torch.from_numpy(b.rho).pin_memory()
    L3 = torch.empty((frames, cfg.N, cfg.q), dtype=torch.float32).pin_memory()
    st3 = torch.empty(frames, dtype=torch.int32).pin_memory()
    d.decode_host(rx, off, rho, None, L3, st3)
    np.testing.assert_array_equal(st3.numpy(), st1)
    np.testing.assert_allclose(L3.numpy(), L1, rtol=1e-5, atol=1e-30)
    picks = [0, frames // 2, frames - 1]
    assert_parity(L3.numpy().astype(np.float64), st3.numpy(), run_oracle(cfg, b, picks), picks)


@pytest.mark.parametrize("name,frames", [("C2", 37), ("C3", 5)])
def test_alpha_beta_overlap_subbatches_bit_identical(name, frames, monkeypatch):
    """The alpha/beta-overlapped sub-batch pipeline (side stream) changes only
    the launch order: every frame's arithmetic is the same, so L must be bit-identical to the
    single-stream schedule, and still match the oracle."""
    cfg = small_cfg(name)
    b = bsidgen.make_batch(cfg, 11, frames)
    outs = []
    for sub in ("1", "3", "4"):
        monkeypatch.setenv("BSIDMAP_AB_SUB", sub)
        d, L, st = run_gpu(cfg, b, 3)
        assert d.plan(frames)["alpha_beta_overlap_subbatches"] == min(int(sub), frames)
        outs.append((L, st))
    for L, st in outs[1:]:
        np.testing.assert_array_equal(st, outs[0][1])
        np.testing.assert_array_equal(L, outs[0][0])
    assert_parity(outs[1][0], outs[1][1], run_oracle(cfg, b, range(3)), range(3))


@pytest.mark.parametrize("name,frames", [("C1", 9), ("C2", 7), ("C4", 2), ("C3", 3), ("C5r", 2)])
def test_app_two_folded_rows(name, frames, monkeypatch):
    """APP pass with the last TWO lattice rows folded into its weights (row n-1 transposed,
    SpecCoreX2::row_transpose; C4's row n-1 has structurally-zero and column-0 nodes) against the
    oracle and the one-row fold."""
    if name == "C5r":  # C5's shape (scalar core, priors) with N cut for the oracle
        full = bsidgen.configs()["C5"]
        cfg = small_cfg("C5", N=40, mn=full.mn, mt=full.mt)
    else:
        cfg = small_cfg(name)
    b = bsidgen.make_batch(cfg, 5, frames)
    monkeypatch.setenv("BSIDMAP_APP_KS", "2")
    d2, L2, st2 = run_gpu(cfg, b, 3)
    assert d2.plan(frames)["app_folded_rows"] == 2
    monkeypatch.setenv("BSIDMAP_APP_KS", "1")
    d1, L1, st1 = run_gpu(cfg, b, 3)
    assert d1.plan(frames)["app_folded_rows"] == 1
    monkeypatch.delenv("BSIDMAP_APP_KS")
    auto = _dec().from_config(cfg, b.C, mode=3, device=0).plan(frames)["app_folded_rows"]
    # one folded row on the pair core (C1, C2, C4), two on the scalar APP core (C3, C5)
    assert auto == (1 if name in ("C1", "C2", "C4") else 2)
    np.testing.assert_array_equal(st2, st1)
    np.testing.assert_allclose(L2, L1, rtol=2e-5, atol=1e-30)
    assert_parity(L2, st2, run_oracle(cfg, b))


def test_modes_agree_and_plan(monkeypatch):
    cfg = small_cfg("C2")
    b = bsidgen.make_batch(cfg, 0, 16)
    _, Ls, sts = run_gpu(cfg, b, 1)
    d, Lr, str_ = run_gpu(cfg, b, 2)
    _, Lg, stg = run_gpu(cfg, b, 3)
    np.testing.assert_array_equal(sts, str_)
    np.testing.assert_array_equal(sts, stg)
    np.testing.assert_allclose(Ls, Lr, rtol=2e-5, atol=1e-30)
    np.testing.assert_allclose(Lg, Lr, rtol=2e-5, atol=1e-30)
    # RECOMPUTE on a spec core: the slab schedule (Gamma for two slabs of symbol indices, alpha and
    # beta rows); memory estimate at the bench batch: stored gamma > Gamma-sum > slab
    assert d.plan(65536)["mode"] == "recompute-slab" and d.plan(64)["core"] == "spec"
    assert _dec().from_config(cfg, b.C, mode=0, device=0).plan(64)["mode"] == "recompute-gammasum"
    assert d.workspace_bytes(65536, 1) > d.workspace_bytes(65536, 3) > 3 * d.workspace_bytes(65536, 2)
    # BSIDMAP_SLAB=0: the paper's per-frame local kernels (alpha rows only), one warp per frame for
    # M_tau <= 64 and one CTA per frame above; AUTO the Gamma-sum schedule
    monkeypatch.setenv("BSIDMAP_SLAB", "0")
    dl, Ll, stl = run_gpu(cfg, b, 2)
    assert dl.plan(65536)["mode"] == "recompute-local"
    np.testing.assert_array_equal(stl, stg)
    np.testing.assert_allclose(Ll, Lr, rtol=2e-5, atol=1e-30)
    assert d.workspace_bytes(16, 1) > d.workspace_bytes(16, 3) > dl.workspace_bytes(16, 2)
    assert dl.workspace_bytes(16, 2) < 16 * (cfg.N + 1) * cfg.Mt * 8 + 512
    c3 = small_cfg("C3")
    d3 = _dec().from_config(c3, bsidgen.codebook(c3), mode=2, device=0)
    assert d3.plan(8)["mode"] == "recompute-local-cta"
    assert d3.workspace_bytes(8, 2) < 8 * (c3.N + 1) * c3.Mt * 8 + 512
    monkeypatch.delenv("BSIDMAP_SLAB")
    assert _dec().from_config(c3, bsidgen.codebook(c3), mode=2, device=0).plan(8)["mode"] == "recompute-slab"
    assert _dec().from_config(c3, bsidgen.codebook(c3), mode=0, device=0).plan(8)["mode"] == "recompute-gammasum"


def test_alpha_beta_states_vs_oracle():
    cfg = small_cfg("C2")
    b = bsidgen.make_batch(cfg, 0, 3)
    d, L, st = run_gpu(cfg, b, 3)
    a, be = d.debug_states(3)
    a, be = a.cpu().numpy(), be.cpu().numpy()
    res = [oracle.decode(oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt),
                         b.bits(f), want_states=True) for f in range(3)]
    for f in range(3):
        for name, g in (("alpha", a[f]), ("beta", be[f])):
            o = res[f][name]
            big = o > 1e-12
            np.testing.assert_allclose(g[big], o[big], rtol=1e-4)
            assert np.all(np.abs(g[~big] - o[~big]) <= 1e-4 * 1e-12 + 1e-16)


def test_full_c5_frame_properties(monkeypatch):
    """Full-size C5 frames (N = 10^4, tau = 120000): the oracle cannot decode them in
    seconds, so check properties that hold at any size: status OK, rows sum to 1,
    APP calibration (among symbols decided with max_D L > 1 - eps the error rate is
    at most ~eps), and bit-complement symmetry (Q-dot depends only on equality and
    inserted bits are uniform) -- complementing every codeword and every
    received bit must leave L unchanged."""
    if os.environ.get("BSIDMAP_SKIP_LARGE"):
        pytest.skip("large test disabled")
    cfg = small_cfg("C5")
    b = bsidgen.make_batch(cfg, 0, 2)
    d, L, st = run_gpu(cfg, b, 0)
    assert d.plan(2)["mode"] == "recompute-gammasum"
    assert (st == 0).all()
    np.testing.assert_allclose(L.sum(2), 1.0, atol=1e-5)
    conf = L.max(2) > 1 - 1e-3
    wrong = (np.argmax(L, 2) != b.msg) & conf
    assert conf.mean() > 0.5
    assert wrong.sum() <= 1e-3 * conf.sum() + 10
    # complement symmetry
    mask = (1 << cfg.n) - 1
    b2 = bsidgen.Batch(cfg, b.first, (~b.C) & mask, b.msg, b.rx.copy(), b.rho, b.offsets, b.priors, 0)
    for f in range(2):
        bits = 1 - b.bits(f)
        b2.rx[f] = bsidgen.pack_bits(bits, b.rx.shape[1])
    _, L2, st2 = run_gpu(cfg, b2, 0)
    assert (st2 == 0).all()
    np.testing.assert_allclose(L2, L, rtol=1e-5, atol=1e-30)
    # the memory-reduced schedules on the same full-size frames agree with the Gamma-sum one: the
    # slab schedule (RECOMPUTE's default on the spec cores) and the paper's per-frame local schedule
    # (one CTA per frame, gamma recomputed in the alpha pass and in the combined beta + L pass,
    # P:483-627)
    d3, L3, st3 = run_gpu(cfg, b, 2)
    assert d3.plan(2)["mode"] == "recompute-slab"
    monkeypatch.setenv("BSIDMAP_SLAB", "0")
    d4, L4, st4 = run_gpu(cfg, b, 2)
    assert d4.plan(2)["mode"] == "recompute-local-cta"
    big = L > 1e-20
    for Lx, sx in ((L3, st3), (L4, st4)):
        np.testing.assert_array_equal(sx, st)
        np.testing.assert_allclose(Lx[big], L[big], rtol=2e-4)


# ----------------------------------------------- bench launch configuration, full sizes

@pytest.mark.parametrize("name,frames,picks", [
    ("C2", 65536, [0, 1, 31, 4097, 16383, 16384, 32768, 40000, 50001, 65534, 65535]),
    ("C3", 2048, [0, 1, 63, 64, 511, 1023, 1024, 1500, 2046, 2047]),
    ("C4", 512, [0, 1, 31, 32, 255, 256, 400, 510, 511]),
])
def test_bench_batch_sampled_parity(name, frames, picks):
    """The bench's per-GPU batch (C2: bench.py's default launch, one decode_batch of 65536
    frames; C3/C4: the 8-GPU configs' per-GPU batch) decoded in ONE call, and frames sampled
    across it (first/last, tile, warp, sub-batch and chunk boundaries) checked one by one
    against the FP64 oracle at the north-star tolerance."""
    if os.environ.get("BSIDMAP_SKIP_LARGE"):
        pytest.skip("large test disabled")
    cfg = small_cfg(name)
    b = bsidgen.make_batch(cfg, 0, frames)
    d, L, st = run_gpu(cfg, b, 0)
    assert (st == 0).all()
    np.testing.assert_allclose(L.sum(2), 1.0, atol=1e-5)
    threads = os.cpu_count() or 1
    oracle.set_threads(max(1, threads // len(picks)))   # long frames: threads inside each frame too
    try:
        assert_parity(L, st, run_oracle(cfg, b, picks), picks)
    finally:
        oracle.set_threads(1)


@pytest.mark.slow
def test_full_c5_frame_vs_oracle(monkeypatch):
    """BASELINE's C5 at full length (q=64, n=12, N=10^4, tau=120000, Pi=Pd=0.02, non-uniform
    priors), decoded end to end on the GPU and compared element by element with the FP64 oracle
    (eqn:L) at the north-star gate: max relative error 1e-4 on every L_i(D), hard
    decisions equal where the oracle's top-two gap exceeds 1e-3.  The GPU decodes the C5 per-GPU
    batch of the 8-GPU config (32 frames) three ways: AUTO with the default geometry (Gamma-sum,
    alpha/beta overlapped on two sub-batches), AUTO chunked in two by a workspace limit (the checked
    frame sits in the second chunk), RECOMPUTE (the slab schedule) and RECOMPUTE with
    BSIDMAP_SLAB=0 (the paper's per-frame local schedule).  The
    oracle decodes the checked frame with its m' loops on every host core (bit-identical to the
    serial oracle, test_threaded_oracle_bit_identical) while the GPU runs."""
    import threading
    cfg = small_cfg("C5")
    frames, pick = 32, 21
    b = bsidgen.make_batch(cfg, 0, frames)
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    box = {}

    def run():
        oracle.set_threads(os.cpu_count() or 1)
        try:
            box["r"] = oracle.decode(prob, b.bits(pick), b.priors[pick].astype(np.float64))
        finally:
            oracle.set_threads(1)

    th = threading.Thread(target=run)
    th.start()
    runs = {}
    d, L, st = run_gpu(cfg, b, 0)
    assert d.plan(frames)["mode"] == "recompute-gammasum"
    runs["auto"] = (L, st)
    per = d.workspace_bytes(1, 3)
    d2, L2, st2 = run_gpu(cfg, b, 0, ws_limit=per * 16 + per // 2)
    assert d2.plan(frames)["chunks"] == 2
    runs["auto-chunked"] = (L2, st2)
    d3, L3, st3 = run_gpu(cfg, b, 2)
    assert d3.plan(frames)["mode"] == "recompute-slab"
    runs["recompute-slab"] = (L3, st3)
    monkeypatch.setenv("BSIDMAP_SLAB", "0")
    d4, L4, st4 = run_gpu(cfg, b, 2)
    assert d4.plan(frames)["mode"] == "recompute-local-cta"
    runs["recompute-local"] = (L4, st4)
    th.join()
    r = box["r"]
    assert r["status"] == oracle.OK
    for name, (Lg, sg) in runs.items():
        assert (sg == 0).all(), name
        w = assert_parity(Lg[pick:pick + 1], sg[pick:pick + 1], [r])
        print(f"C5 full frame {pick}, {name}: max rel err {w:.3e}")


def test_decode_captures_into_cuda_graph():
    """decode_batch is stream-ordered and allocation-free once its workspace exists, so a caller
    can capture it in a CUDA graph and replay it (launch-bound small batches: C1 latency); the
    replayed result equals the eager one bit for bit."""
    cfg = small_cfg("C1")
    b = bsidgen.make_batch(cfg, 3, 4)
    Decoder = _dec()
    d = Decoder.from_config(cfg, b.C, device=0)
    rx, off, rho, pri = to_dev(b)
    L = torch.empty((4, cfg.N, cfg.q), dtype=torch.float32, device="cuda")
    st = torch.empty((4,), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d.decode_batch(rx, off, rho, pri, L, st, s)   # warm-up: workspace, smem opt-ins
    torch.cuda.synchronize()
    L_eager = L.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        d.decode_batch(rx, off, rho, pri, L, st, s)
    L.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(L, L_eager)
    assert (st == 0).all()


# ------------------------------------------------------- live-window APP (k_live + k_app_live_*)

def _cfg_n(name, N):
    import dataclasses
    cfg = bsidgen.configs()[name]
    return cfg if N is None else dataclasses.replace(cfg, N=N)


@pytest.mark.parametrize("name,N,frames,G", [
    ("C1", None, 300, None), ("C2", None, 400, None), ("C2", None, 37, 3), ("C2", None, 9, 16),
    ("C3", 40, 5, 2), ("C4", 30, 3, None), ("C5", 30, 5, 4), ("C5", 30, 3, 1)])
def test_live_window_app(name, N, frames, G, monkeypatch):
    """The APP over live windows only (reading R18): k_live marks each (frame, i) row's
    windows with posterior mass above eps = 2^-128 of the row's, k_app_live_* packs G frames per
    warp and walks their live windows in rounds.  Against the FP64 oracle at the north-star gate,
    and with eps = 0 (exactly-zero windows skipped only).
    G = 16 with 9 frames: one warp, frames of every round count; 400 C2 frames: the automatic G."""
    cfg = _cfg_n(name, N)
    b = bsidgen.make_batch(cfg, 40, frames)
    if G is not None:
        monkeypatch.setenv("BSIDMAP_APP_G", str(G))
    d, L, st = run_gpu(cfg, b, 3)
    pl = d.plan(frames)
    assert pl["app_live"] == 1 and pl["mode"] == "recompute-gammasum"
    if G is not None:
        assert pl["app_frames_per_warp"] == G
    res = run_oracle(cfg, b)
    assert_parity(L, st, res)
    monkeypatch.setenv("BSIDMAP_LIVE_EPS", "0")
    _, L0, st0 = run_gpu(cfg, b, 3)
    assert_parity(L0, st0, res)
    np.testing.assert_array_equal(st, st0)
    # every L entry moves by at most M_tau eps (reading R18) between the two thresholds
    assert np.abs(L - L0).max() <= max(1e-6, cfg.Mt * 2.0 ** -128)


def test_live_window_app_mixed_status(monkeypatch):
    """Frames whose end drift is out of range (status DRIFT_OUT_OF_RANGE: no live windows, zero L
    rows) sit between OK frames of one warp's G = 8 frames, on the C1 spec shape."""
    cfg = small_cfg("C1")
    F = 19
    b = bsidgen.make_batch(cfg, 0, F)
    b.rx = np.concatenate([b.rx, np.zeros((F, 2), np.uint32)], 1)
    b.offsets = np.arange(F, dtype=np.int64) * b.rx.shape[1]
    for f, dm in ((3, cfg.mt[1] + 1), (7, cfg.mt[0] - 1), (8, cfg.mt[1] + 2), (18, cfg.mt[0] - 2)):
        b.rho[f] = cfg.tau + dm
    monkeypatch.setenv("BSIDMAP_APP_G", "8")
    d, L, st = run_gpu(cfg, b, 3)
    assert d.plan(F)["app_live"] == 1 and d.plan(F)["app_frames_per_warp"] == 8
    res = run_oracle(cfg, b)
    assert [int(st[f]) for f in (3, 7, 8, 18)] == [1, 1, 1, 1]
    assert_parity(L, st, res)


@pytest.mark.parametrize("name,N,frames", [("C2", None, 61), ("C5", 24, 9), ("C3", 30, 7)])
def test_live_app_independent_of_packing(name, N, frames, monkeypatch):
    """The frames per warp G only changes how a frame's live windows are packed into rounds (and so
    the FP64 association of a frame split over two rounds): L is the same for every G -- bit-identical
    after the FP32 rounding of the output in practice, gated here at 1e-12 relative."""
    cfg = _cfg_n(name, N)
    b = bsidgen.make_batch(cfg, 7, frames)
    outs = []
    for G in (1, 3, 5, 12, 16):
        monkeypatch.setenv("BSIDMAP_APP_G", str(G))
        d, L, st = run_gpu(cfg, b, 3)
        assert d.plan(frames)["app_frames_per_warp"] == G
        outs.append((L, st))
    for L, st in outs[1:]:
        np.testing.assert_array_equal(st, outs[0][1])
        np.testing.assert_allclose(L, outs[0][0], rtol=1e-12, atol=0)
