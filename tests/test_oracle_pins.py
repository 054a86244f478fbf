"""Pins for the FP64 oracle (oracle/), checked against things other than itself:
SPEC worked values (tests/golden/spec_examples.txt), brute-force enumeration of
channel event sequences (tests/brute.py), exhaustive Bayes over messages,
closed forms and invariants.  CPU only."""
import itertools
import math
import os

import numpy as np
import pytest

import bsidgen
import oracle
from tests import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


def _golden():
    rows = []
    for line in open(GOLDEN):
        line = line.split("#")[0].strip()
        if line:
            rows.append(line.split())
    return rows


# ---------------------------------------------------------------- SPEC values

def test_spec_qdot_values():
    rows = [r for r in _golden() if r[0] == "qdot"]
    assert len(rows) == 3
    for _, y, x, Pi, Pd, Ps, exp, *_ in rows:
        got = oracle.qdot(int(y), int(x), float(Pi), float(Pd), float(Ps))
        assert got == pytest.approx(float(exp), rel=1e-15, abs=1e-300)


def test_spec_lattice_last_row():
    rows = [r for r in _golden() if r[0] == "lattice_last_row"]
    assert rows
    for _, x, y, Pi, Pd, Ps, lo, hi, exp, *_ in rows:
        xb = [int(c) for c in x]
        yb = [int(c) for c in y]
        F = oracle.lattice(xb, yb, float(Pi), float(Pd), float(Ps), corridor=(int(lo), int(hi)))
        expected = [float(v) for v in exp.split(",")]
        np.testing.assert_allclose(F[len(xb), :], expected, rtol=1e-14)


def test_spec_drift_pmf_values():
    for _, T, Pi, Pd, exp, *_ in [r for r in _golden() if r[0] == "drift_pmf"]:
        off, p = bsidgen.drift_pmf(int(T), float(Pi), float(Pd))
        for item in exp.split(","):
            d, v = item.split(":")
            assert p[int(d) - off] == pytest.approx(float(v), rel=1e-12)


# ------------------------------------------------------- lattice vs brute force

def test_receiver_closed_forms():
    # R(()|x) = Pd^n when Pi = 0 (only the all-delete path)
    for n in range(1, 6):
        x = [1, 0, 1, 1, 0][:n]
        assert oracle.receiver(x, [], 0.0, 0.3, 0.0) == pytest.approx(0.3 ** n, rel=1e-14)
    # noiseless: R(x|x) = 1, R(y|x) = 0 for y != x
    x = [1, 0, 0, 1, 1, 1]
    assert oracle.receiver(x, x, 0.0, 0.0, 0.0) == 1.0
    assert oracle.receiver(x, [1, 0, 0, 1, 1, 0], 0.0, 0.0, 0.0) == 0.0
    # substitution only: Ps^dH (1-Ps)^(n-dH)
    y = [0, 0, 0, 1, 1, 0]
    dh = sum(a != b for a, b in zip(x, y))
    assert oracle.receiver(x, y, 0.0, 0.0, 0.1) == pytest.approx(0.1 ** dh * 0.9 ** (6 - dh), rel=1e-14)


@pytest.mark.parametrize("seed", range(6))
def test_lattice_equals_event_enumeration(seed):
    rng = np.random.default_rng(1000 + seed)
    worst = 0.0
    for _ in range(40):
        n = int(rng.integers(1, 5))
        mu = int(rng.integers(0, 9))
        x = rng.integers(0, 2, n)
        y = rng.integers(0, 2, mu)
        Pi, Pd = [float(v) for v in rng.choice([0.0, 0.05, 0.2], 2)]
        Ps = float(rng.choice([0.0, 0.1]))
        corr = None
        if rng.random() < 0.6:
            lo = -int(rng.integers(0, n + 1))
            corr = (lo, int(rng.integers(0, 5)))
        F = oracle.lattice(x, y, Pi, Pd, Ps, corridor=corr)
        # every node of the last row is R(y_1..y_j | x) under the same corridor
        for j in range(mu + 1):
            want = brute.receiver_enum(x, y[:j], Pi, Pd, Ps, corridor=corr)
            got = F[n, j]
            if want == 0.0:
                assert got == 0.0
            else:
                worst = max(worst, abs(got - want) / want)
    assert worst < 1e-12


def test_lattice_column_sums_equal_drift_pmf():
    """sum over all y of length l of R(y|x) = P(S_n = l - n) (unconstrained)."""
    Pi, Pd, Ps = 0.15, 0.1, 0.05
    for n in (1, 2, 3):
        x = [1, 0, 1][:n]
        off, pmf = bsidgen.drift_pmf(n, Pi, Pd)
        for l in range(0, 2 * n + 3):
            s = sum(oracle.receiver(x, list(y), Pi, Pd, Ps) for y in itertools.product([0, 1], repeat=l))
            want = pmf[l - n - off] if 0 <= l - n - off < len(pmf) else 0.0
            assert s == pytest.approx(want, rel=1e-12, abs=1e-300)


# ------------------------------------------------------------ full decoder pins

def _tiny_problem(rng, wide=False):
    n = int(rng.integers(1, 4))
    q = int(rng.integers(2, min(4, 2 ** n) + 1))
    N = int(rng.integers(1, 4))
    while n * N > 6:
        N -= 1
    N = max(N, 1)
    C = np.array([rng.choice(2 ** n, q, replace=False) for _ in range(N)], dtype=np.uint32)
    Pi, Pd = [float(v) for v in rng.choice([0.0, 0.05, 0.2], 2)]
    if Pi + Pd == 0:
        Pi = 0.1
    Ps = float(rng.choice([0.0, 0.1]))
    tau = n * N
    if wide:
        mn = (-n, tau + 3)
        mt = (-tau, tau + 3)
    else:
        mn = (-int(rng.integers(0, n + 1)), int(rng.integers(0, 3)))
        mt = (mn[0] - int(rng.integers(0, 3)), mn[1] + int(rng.integers(0, 3)))
    # received sequence: channel output of a random message, length kept inside mt
    msg = rng.integers(0, q, N)
    X = bsidgen.encode(C, msg, n)
    for _ in range(100):
        Y = []
        for b in X:
            while True:
                u = rng.random()
                if u < Pi:
                    Y.append(int(rng.integers(0, 2)))
                    continue
                if u >= Pi + Pd:
                    Y.append(int(b) ^ int(rng.random() < Ps))
                break
        if mt[0] <= len(Y) - tau <= mt[1]:
            break
    priors = None
    if rng.random() < 0.4:
        priors = rng.random((N, q)) + 0.05
        priors /= priors.sum(1, keepdims=True)
    prob = oracle.Problem(q, n, N, C, Pi, Pd, Ps, mn, mt)
    return prob, np.array(Y, dtype=np.uint8), priors


@pytest.mark.parametrize("seed", range(12))
def test_decoder_equals_exhaustive_bayes(seed):
    rng = np.random.default_rng(seed)
    checked = 0
    for trial in range(6):
        prob, Y, priors = _tiny_problem(rng, wide=(trial % 3 == 0))
        if not (prob.mt_lo <= len(Y) - prob.n * prob.N <= prob.mt_hi):
            continue
        res = oracle.decode(prob, Y, priors, want_states=True)
        Lb, ev = brute.posterior_enum(prob.C.tolist(), prob.n, Y.tolist(), prob.Pi, prob.Pd, prob.Ps,
                                      priors.tolist() if priors is not None else None,
                                      (prob.mn_lo, prob.mn_hi), (prob.mt_lo, prob.mt_hi))
        if ev == 0.0:
            assert res["status"] == oracle.UNDERFLOW
            continue
        assert res["status"] == oracle.OK
        np.testing.assert_allclose(res["L"], np.array(Lb), rtol=0, atol=1e-9)
        # ln lambda_N(rho - tau) = ln P(Y) under the constraints (eqn:L normaliser)
        assert res["log_lambda"] == pytest.approx(math.log(ev), rel=1e-10, abs=1e-10)
        checked += 1
    assert checked >= 2


def test_wide_limits_equal_unconstrained_posterior():
    rng = np.random.default_rng(77)
    for _ in range(8):
        prob, Y, priors = _tiny_problem(rng, wide=True)
        res = oracle.decode(prob, Y, priors)
        Lb, ev = brute.posterior_enum(prob.C.tolist(), prob.n, Y.tolist(), prob.Pi, prob.Pd, prob.Ps,
                                      priors.tolist() if priors is not None else None, None, None)
        assert ev > 0
        assert res["status"] == oracle.OK
        np.testing.assert_allclose(res["L"], np.array(Lb), rtol=0, atol=1e-9)


def _frame(cfg_name="C1", f=0, **over):
    cfg = bsidgen.configs()[cfg_name]
    for k, v in over.items():
        setattr(cfg, k, v)
    b = bsidgen.make_batch(cfg, f, 1)
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    return cfg, b, prob


def test_normaliser_and_lambda_constancy():
    """sum_D L_i(D) = 1 with the LITERAL 1/lambda_N, and
    sum_m alpha_i(m) beta_i(m) = lambda_N for every i (eqn:lambda)."""
    for f in range(3):
        cfg, b, prob = _frame("C1", f)
        res = oracle.decode(prob, b.bits(0), want_states=True)
        assert res["status"] == oracle.OK
        np.testing.assert_allclose(res["L"].sum(1), 1.0, rtol=0, atol=1e-12)
        lam = [math.log((res["alpha"][i] * res["beta"][i]).sum()) + res["logA"][i] + res["logB"][i]
               for i in range(cfg.N + 1)]
        np.testing.assert_allclose(lam, res["log_lambda"], rtol=0, atol=1e-12)


def test_noiseless_point_mass():
    cfg, b, prob = _frame("C1", 0, Pi=0.0, Pd=0.0, Ps=0.0, mn=(0, 0), mt=(0, 0))
    res = oracle.decode(prob, b.bits(0))
    assert res["status"] == oracle.OK
    L = res["L"]
    for i, D in enumerate(b.msg[0]):
        assert L[i, D] == pytest.approx(1.0, abs=1e-13)
        assert L[i].sum() == pytest.approx(1.0, abs=1e-13)


def test_substitution_only_closed_form():
    cfg, b, prob = _frame("C1", 0, Pi=0.0, Pd=0.0, Ps=0.07, mn=(0, 0), mt=(0, 0))
    pri = np.random.default_rng(5).random((cfg.N, cfg.q)) + 0.1
    res = oracle.decode(prob, b.bits(0), pri)
    Y = b.bits(0)
    for i in range(cfg.N):
        seg = Y[i * cfg.n:(i + 1) * cfg.n]
        w = np.array([pri[i, D] * np.prod([0.07 if ((int(b.C[i, D]) >> t) & 1) != seg[t] else 0.93
                                           for t in range(cfg.n)]) for D in range(cfg.q)])
        np.testing.assert_allclose(res["L"][i], w / w.sum(), rtol=1e-13)


def test_single_symbol_direct_bayes():
    """N=1: L_0(D) proportional to P(D) R(Y|C_0(D)), R by enumeration."""
    rng = np.random.default_rng(9)
    for _ in range(5):
        n, q = 3, 4
        C = np.array([rng.choice(8, q, replace=False)], dtype=np.uint32)
        Y = rng.integers(0, 2, int(rng.integers(2, 5))).astype(np.uint8)
        prob = oracle.Problem(q, n, 1, C, 0.1, 0.15, 0.05, (-3, 3), (-3, 3))
        pri = rng.random(q) + 0.1
        res = oracle.decode(prob, Y, pri.reshape(1, q))
        w = np.array([pri[D] * brute.receiver_enum([(int(C[0, D]) >> t) & 1 for t in range(n)], Y,
                                                   0.1, 0.15, 0.05, corridor=(-3, 3)) for D in range(q)])
        np.testing.assert_allclose(res["L"][0], w / w.sum(), rtol=1e-12)


def test_prior_invariances():
    cfg, b, prob = _frame("C1", 1)
    base = oracle.decode(prob, b.bits(0))["L"]
    rng = np.random.default_rng(3)
    # scaling a prior row leaves L unchanged (uniform priors x 7)
    res = oracle.decode(prob, b.bits(0), np.full((cfg.N, cfg.q), 7.0 / cfg.q))
    np.testing.assert_allclose(res["L"], base, rtol=1e-12)
    # one-hot prior forces L = 1 there
    pri = rng.random((cfg.N, cfg.q)) + 0.1
    pri[4] = 0
    pri[4, 3] = 1.0
    res = oracle.decode(prob, b.bits(0), pri)
    assert res["L"][4, 3] == pytest.approx(1.0, abs=1e-14)


def test_bit_complement_symmetry():
    """Complementing every codeword and every received bit leaves L unchanged:
    Q-dot depends only on equality and inserted bits are uniform."""
    cfg, b, prob = _frame("C1", 2)
    mask = (1 << cfg.n) - 1
    prob2 = oracle.Problem(cfg.q, cfg.n, cfg.N, (~b.C) & mask, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    L1 = oracle.decode(prob, b.bits(0))["L"]
    L2 = oracle.decode(prob2, 1 - b.bits(0))["L"]
    np.testing.assert_array_equal(L1, L2)


def test_drift_out_of_range_and_underflow_status():
    cfg, b, prob = _frame("C1", 0)
    Y = b.bits(0)
    too_long = np.concatenate([Y, np.zeros(cfg.mt[1] - (len(Y) - cfg.tau) + 1, np.uint8)])
    res = oracle.decode(prob, too_long)
    assert res["status"] == oracle.DRIFT_OUT_OF_RANGE
    assert not res["L"].any()
    # noiseless channel, wrong received bits -> no path: underflow
    prob0 = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, 0.0, 0.0, 0.0, (0, 0), (0, 0))
    bad = np.ones(cfg.tau, np.uint8)
    # make sure no codeword of position 0 is all ones
    if any(int(w) == (1 << cfg.n) - 1 for w in b.C[0]):
        bad[0] = 0
    res = oracle.decode(prob0, bad)
    assert res["status"] in (oracle.UNDERFLOW, oracle.OK)
    if not any(all(((int(w) >> t) & 1) == bad[t] for t in range(cfg.n)) for w in b.C[0]):
        assert res["status"] == oracle.UNDERFLOW


def test_gamma_entries_equal_enumeration():
    """gamma_i(m', m, D) = P(D) R(Y[ni+m' .. n(i+1)+m) | C_i(D)) (eqn:gamma),
    R by event enumeration with the corridor, zero outside the windows."""
    cfg, b, prob = _frame("C1", 0)
    Y = b.bits(0)
    rho = len(Y)
    for i in (0, 4, cfg.N - 1):
        g = oracle.gamma(prob, Y, i)
        for mp in range(cfg.mt[0], cfg.mt[1] + 1, 3):
            for k in range(cfg.mn[0], cfg.mn[1] + 1):
                m = mp + k
                for D in (0, cfg.q - 1):
                    s, e = cfg.n * i + mp, cfg.n * (i + 1) + m
                    got = g[mp - cfg.mt[0], k - cfg.mn[0], D]
                    if s < 0 or s > rho or e > rho or e < s or not (cfg.mt[0] <= m <= cfg.mt[1]):
                        assert got == 0.0
                        continue
                    x = [(int(b.C[i, D]) >> t) & 1 for t in range(cfg.n)]
                    want = brute.receiver_enum(x, Y[s:e], cfg.Pi, cfg.Pd, cfg.Ps, corridor=cfg.mn) / cfg.q
                    assert got == pytest.approx(want, rel=1e-10, abs=1e-300)


def test_drift_limits_cover_pr():
    for cfg in bsidgen.configs().values():
        for T, (lo, hi) in ((cfg.n, cfg.mn),):
            off, p = bsidgen.drift_pmf(T, cfg.Pi, cfg.Pd)
            outside = p[: max(lo - off, 0)].sum() + p[hi - off + 1:].sum()
            assert outside <= 1e-10
    # drift PMF moments: mean (Pi - Pd)/(1 - Pi) per bit (closed form of the geometric insertion count)
    off, p = bsidgen.drift_pmf(50, 0.1, 0.05)
    d = np.arange(len(p)) + off
    assert (p * d).sum() == pytest.approx(50 * (0.1 - 0.05) / (1 - 0.1), rel=1e-9)


# ------------------------------------------- NEXT-1 / NEXT-4 oracle extensions

def test_soft_boundary_priors_equal_exhaustive_bayes():
    """alpha_0 / beta_N as distributions over drift states (Phi_T): the
    oracle equals Bayes over messages x start offsets x event sequences x end drifts."""
    rng = np.random.default_rng(21)
    checked = 0
    for trial in range(14):
        prob, Y, priors = _tiny_problem(rng, wide=(trial % 2 == 0))
        # pad the received sequence with random bits that no frame bit explains
        Y = np.concatenate([rng.integers(0, 2, int(rng.integers(0, 3))), Y,
                            rng.integers(0, 2, int(rng.integers(0, 3)))]).astype(np.uint8)
        Mt = prob.Mt
        a0 = rng.random(Mt) * (rng.random(Mt) < 0.6)
        a0[0 - prob.mt_lo] += 0.3
        bN = rng.random(Mt)
        res = oracle.decode(prob, Y, priors, alpha0=a0, betaN=bN)
        states = range(prob.mt_lo, prob.mt_hi + 1)
        Lb, ev = brute.posterior_soft(prob.C.tolist(), prob.n, Y.tolist(), prob.Pi, prob.Pd, prob.Ps,
                                      priors.tolist() if priors is not None else None,
                                      (prob.mn_lo, prob.mn_hi), (prob.mt_lo, prob.mt_hi),
                                      {m: a0[m - prob.mt_lo] for m in states}, {m: bN[m - prob.mt_lo] for m in states})
        if ev == 0.0:
            assert res["status"] == oracle.UNDERFLOW
            continue
        assert res["status"] == oracle.OK
        np.testing.assert_allclose(res["L"], np.array(Lb), rtol=0, atol=1e-9)
        assert res["log_lambda"] == pytest.approx(math.log(ev), rel=1e-10, abs=1e-10)
        checked += 1
    assert checked >= 6


def test_point_mass_boundaries_reduce_to_default():
    cfg, b, prob = _frame("C1", 3)
    Y = b.bits(0)
    base = oracle.decode(prob, Y)
    a0 = np.zeros(prob.Mt)
    a0[-prob.mt_lo] = 2.0
    bN = np.zeros(prob.Mt)
    bN[len(Y) - cfg.tau - prob.mt_lo] = 5.0
    soft = oracle.decode(prob, Y, alpha0=a0, betaN=bN)
    np.testing.assert_allclose(soft["L"], base["L"], rtol=1e-13)


def test_extrinsic_equals_posterior_without_own_prior():
    """E_i(D) proportional to L_i(D)/P(D_i=D) equals the exhaustive
    Bayes posterior of D_i computed with row i of the priors replaced by uniform."""
    rng = np.random.default_rng(33)
    for _ in range(5):
        prob, Y, _ = _tiny_problem(rng, wide=True)
        pri = rng.random((prob.N, prob.q)) + 0.05
        res = oracle.decode(prob, Y, pri, extrinsic=True)
        for i in range(prob.N):
            mod = pri.copy()
            mod[i] = 1.0
            Lb, ev = brute.posterior_enum(prob.C.tolist(), prob.n, Y.tolist(), prob.Pi, prob.Pd, prob.Ps,
                                          mod.tolist(), (prob.mn_lo, prob.mn_hi), (prob.mt_lo, prob.mt_hi))
            np.testing.assert_allclose(res["E"][i], np.array(Lb[i]), rtol=0, atol=1e-9)
    # zero prior: the extrinsic is 0 there, and E = L under uniform priors
    cfg, b, prob = _frame("C1", 0)
    pri = np.full((cfg.N, cfg.q), 1.0)
    pri[2, 1] = 0.0
    res = oracle.decode(prob, b.bits(0), pri, extrinsic=True)
    assert res["E"][2, 1] == 0.0
    np.testing.assert_allclose(res["E"].sum(1), 1.0, atol=1e-12)
    res_u = oracle.decode(prob, b.bits(0), extrinsic=True)
    np.testing.assert_allclose(res_u["E"], res_u["L"] / res_u["L"].sum(1, keepdims=True), rtol=1e-13)


@pytest.mark.parametrize("threads", [2, 5, 8])
def test_threaded_oracle_bit_identical(threads):
    """oracle.set_threads(t) splits only loops whose iterations are independent (gamma's m' loop,
    L's D loop, beta's m' loop) and keeps every sum's serial order, so the threaded decode must
    equal the single-threaded one bit for bit -- including the states, the log scales, soft
    frame boundaries and non-uniform priors -- and therefore inherits every pin above."""
    import dataclasses
    cfg = dataclasses.replace(bsidgen.configs()["C2"], N=30, priors=True)
    b = bsidgen.make_batch(cfg, 77, 2)
    prob = oracle.Problem(cfg.q, cfg.n, cfg.N, b.C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt)
    rng = np.random.default_rng(threads)
    kw = dict(want_states=True, extrinsic=True)
    for f in range(2):
        args = (prob, b.bits(f), b.priors[f].astype(np.float64))
        extra = {} if f == 0 else dict(alpha0=rng.random(prob.Mt), betaN=rng.random(prob.Mt))
        try:
            oracle.set_threads(1)
            r1 = oracle.decode(*args, **kw, **extra)
            g1 = oracle.gamma(prob, b.bits(f), 17, b.priors[f])
            oracle.set_threads(threads)
            rt = oracle.decode(*args, **kw, **extra)
            gt = oracle.gamma(prob, b.bits(f), 17, b.priors[f])
        finally:
            oracle.set_threads(1)
        assert r1["status"] == rt["status"] == oracle.OK
        assert r1["log_lambda"] == rt["log_lambda"]
        for k in ("L", "E", "alpha", "beta", "logA", "logB"):
            np.testing.assert_array_equal(rt[k], r1[k])
        np.testing.assert_array_equal(gt, g1)
