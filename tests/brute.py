"""Brute-force pins written against the BSID channel's GENERATIVE definition
(P:85-109), never against the lattice recursion, so they are independent of
both the oracle and the CUDA path.

* ``receiver_enum``   -- R(y|x): sum over explicit channel event sequences.
* ``posterior_enum``  -- exhaustive Bayes over all q^N messages x all event
  sequences of the whole frame, with the decoder's state-space constraints
  (drift at codeword boundaries in [m_tau^-, m_tau^+], within-codeword drift
  relative to the codeword's start in [m_n^-, m_n^+]) applied to every
  visited (bits consumed, bits received) node.

Channel events at time t: insertion with probability Pi (a
uniform random bit is output, so matching a given received bit costs
Pi/2; the channel stays at time t), deletion Pd, transmission
Pt = 1 - Pi - Pd with substitution Ps.  No insertion follows the frame's
last bit (eqn:F_lastrow).
"""
from __future__ import annotations

import itertools


def _transmit_prob(ybit, xbit, Pi, Pd, Ps):
    Pt = 1.0 - Pi - Pd
    return Pt * (Ps if ybit != xbit else 1.0 - Ps)


def receiver_enum(x, y, Pi, Pd, Ps, corridor=None):
    """Sum of the probabilities of every event sequence that turns x into exactly y.

    Enumerates sequences explicitly (depth-first, one branch per event); the
    optional corridor (lo, hi) keeps only sequences whose every visited node
    has lo <= received - consumed <= hi.
    """
    x = [int(b) for b in x]
    y = [int(b) for b in y]
    n, mu = len(x), len(y)
    total = 0.0
    stack = [(0, 0, 1.0)]  # (bits consumed r, bits output j, path probability)
    while stack:
        r, j, p = stack.pop()
        if corridor is not None and not (corridor[0] <= j - r <= corridor[1]):
            continue
        if r == n:
            if j == mu:
                total += p
            continue
        # insertion before bit r+1: random bit, must equal y_{j+1}
        if j < mu and Pi > 0:
            stack.append((r, j + 1, p * Pi * 0.5))
        # deletion of bit r+1
        if Pd > 0:
            stack.append((r + 1, j, p * Pd))
        # transmission of bit r+1 as y_{j+1}
        if j < mu:
            t = _transmit_prob(y[j], x[r], Pi, Pd, Ps)
            if t > 0:
                stack.append((r + 1, j + 1, p * t))
    return total


def frame_likelihood_enum(X, Y, n, Pi, Pd, Ps, mn=None, mt=None):
    """P(Y | X) over explicit event sequences of a whole frame (tau = len(X)).

    With mn/mt given, every sequence must keep (a) the drift j - t at each
    codeword boundary node t = n i in [mt_lo, mt_hi], and (b) every node
    visited while codeword i is being sent within [mn_lo, mn_hi] of the
    boundary drift of codeword i (the node reached by bit n(i+1)'s event is
    the last node of codeword i and the first of codeword i+1).
    """
    X = [int(b) for b in X]
    Y = [int(b) for b in Y]
    tau, rho = len(X), len(Y)

    def in_corridor(j, t, d0):
        return mn is None or mn[0] <= (j - t) - d0 <= mn[1]

    def in_frame_limits(j, t):
        return mt is None or mt[0] <= j - t <= mt[1]

    total = 0.0
    stack = [(0, 0, 0, 1.0)]  # (t consumed, j received, start drift of current codeword, prob)
    while stack:
        t, j, d0, p = stack.pop()
        if t == tau:
            if j == rho:
                total += p
            continue
        # insertion before bit t+1: random bit that must equal y_{j+1}; stay at t
        if j < rho and Pi > 0 and in_corridor(j + 1, t, d0):
            stack.append((t, j + 1, d0, p * Pi * 0.5))
        # the event of bit t+1: deletion -> (t+1, j), transmission -> (t+1, j+1)
        events = [(j, Pd)]
        if j < rho:
            events.append((j + 1, _transmit_prob(Y[j], X[t], Pi, Pd, Ps)))
        for nj, pe in events:
            if pe == 0.0:
                continue
            nt = t + 1
            if not in_corridor(nj, nt, d0):
                continue
            nd0 = d0
            if nt % n == 0:  # boundary node: closes this codeword, opens the next
                if not in_frame_limits(nj, nt):
                    continue
                nd0 = nj - nt
            stack.append((nt, nj, nd0, p * pe))
    return total


def posterior_enum(C, n, Y, Pi, Pd, Ps, priors=None, mn=None, mt=None):
    """Exhaustive Bayes: L_i(D) = sum_{msg: D_i = D} P(msg) P(Y|X(msg)) / sum_msg P(msg) P(Y|X(msg)).

    Returns (L [N][q] as nested lists, evidence = sum_msg P(msg) P(Y|X(msg))).
    """
    N, q = len(C), len(C[0])
    num = [[0.0] * q for _ in range(N)]
    evidence = 0.0
    for msg in itertools.product(range(q), repeat=N):
        X = []
        pm = 1.0
        for i, D in enumerate(msg):
            w = int(C[i][D])
            X.extend((w >> t) & 1 for t in range(n))
            pm *= (priors[i][D] if priors is not None else 1.0 / q)
        if pm == 0.0:
            continue
        lik = frame_likelihood_enum(X, Y, n, Pi, Pd, Ps, mn, mt)
        w = pm * lik
        evidence += w
        for i, D in enumerate(msg):
            num[i][D] += w
    if evidence == 0.0:
        return None, 0.0
    return [[v / evidence for v in row] for row in num], evidence


def drift_enum(T, Pi, Pd, kmax=12):
    """P(S_T = m) by enumerating per-bit event tuples (k insertions, then delete or
    transmit) for T bits -- the generative definition of the drift."""
    Pt = 1.0 - Pi - Pd
    per_bit = []
    for k in range(kmax + 1):
        per_bit.append((k - 1, Pi ** k * Pd))
        per_bit.append((k, Pi ** k * Pt))
    out = {}
    for seq in itertools.product(per_bit, repeat=T):
        m = sum(c for c, _ in seq)
        p = 1.0
        for _, w in seq:
            p *= w
        out[m] = out.get(m, 0.0) + p
    return out


def frame_likelihood_soft(X, Y, n, Pi, Pd, Ps, mn, mt, alpha0, betaN):
    """sum_{d0} alpha0(d0) sum_paths P(path) betaN(end drift): the frame's first bit
    enters when d0 received bits precede it and its last bit leaves the channel at any
    received position j <= |Y| (end drift j - tau); bits outside are not explained by
    the frame.  alpha0 / betaN: dicts drift -> weight (frame-boundary priors).
    Same node constraints as frame_likelihood_enum."""
    X = [int(b) for b in X]
    Y = [int(b) for b in Y]
    tau, rho = len(X), len(Y)

    def in_corridor(j, t, d0):
        return mn[0] <= (j - t) - d0 <= mn[1]

    def in_frame_limits(j, t):
        return mt[0] <= j - t <= mt[1]

    total = 0.0
    for start, w0 in alpha0.items():
        if w0 == 0.0 or start < 0 or start > rho or not in_frame_limits(start, 0):
            continue
        stack = [(0, start, start, w0)]
        while stack:
            t, j, d0, p = stack.pop()
            if t == tau:
                total += p * betaN.get(j - tau, 0.0)
                continue
            if j < rho and Pi > 0 and in_corridor(j + 1, t, d0):
                stack.append((t, j + 1, d0, p * Pi * 0.5))
            events = [(j, Pd)]
            if j < rho:
                events.append((j + 1, _transmit_prob(Y[j], X[t], Pi, Pd, Ps)))
            for nj, pe in events:
                if pe == 0.0:
                    continue
                nt = t + 1
                if not in_corridor(nj, nt, d0):
                    continue
                nd0 = d0
                if nt % n == 0:
                    if not in_frame_limits(nj, nt):
                        continue
                    nd0 = nj - nt
                stack.append((nt, nj, nd0, p * pe))
    return total


def posterior_soft(C, n, Y, Pi, Pd, Ps, priors, mn, mt, alpha0, betaN):
    """Exhaustive Bayes with frame-boundary priors; returns (L, evidence)."""
    N, q = len(C), len(C[0])
    num = [[0.0] * q for _ in range(N)]
    evidence = 0.0
    for msg in itertools.product(range(q), repeat=N):
        X = []
        pm = 1.0
        for i, D in enumerate(msg):
            w = int(C[i][D])
            X.extend((w >> t) & 1 for t in range(n))
            pm *= (priors[i][D] if priors is not None else 1.0 / q)
        if pm == 0.0:
            continue
        w = pm * frame_likelihood_soft(X, Y, n, Pi, Pd, Ps, mn, mt, alpha0, betaN)
        evidence += w
        for i, D in enumerate(msg):
            num[i][D] += w
    if evidence == 0.0:
        return None, 0.0
    return [[v / evidence for v in row] for row in num], evidence
