"""FP64 CPU oracle for the BSID MAP decoder of arXiv 1802.08483.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1802_08483_b200``) never imports it, and
the two share no code: this is a ctypes wrapper around ``bsid_oracle.c``
(plain C, FP64, full 2-D lattices, literal 1/lambda_N(rho-tau)), which cites
PAPER.md for every step.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(brute force, closed forms, invariants, SPEC worked values); none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bsid_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libbsid_oracle.so")
_lock = threading.Lock()
_lib = None

OK, DRIFT_OUT_OF_RANGE, UNDERFLOW = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math: IEEE FP64 as written)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            d, i, p = ctypes.c_double, ctypes.c_int, ctypes.c_void_p
            lib.oracle_qdot.restype = d
            lib.oracle_qdot.argtypes = [i, i, d, d, d]
            lib.oracle_lattice.restype = i
            lib.oracle_lattice.argtypes = [i, p, i, p, d, d, d, i, i, i, p]
            lib.oracle_receiver.restype = d
            lib.oracle_receiver.argtypes = [i, p, i, p, d, d, d, i, i, i]
            lib.oracle_decode.restype = i
            lib.oracle_decode.argtypes = [i, i, i, p, d, d, d, i, i, i, i, p, i, p, p, p, p, p, p, p, p, p]
            lib.oracle_extrinsic.restype = i
            lib.oracle_extrinsic.argtypes = [i, i, p, p, p]
            lib.oracle_set_threads.restype = i
            lib.oracle_set_threads.argtypes = [i]
            lib.oracle_gamma_at.restype = i
            lib.oracle_gamma_at.argtypes = [i, i, i, p, d, d, d, i, i, i, i, p, i, p, i, p]
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def qdot(y: int, x: int, Pi: float, Pd: float, Ps: float) -> float:
    return _load().oracle_qdot(int(y), int(x), Pi, Pd, Ps)


def lattice(x, y, Pi, Pd, Ps, corridor=None):
    """Full (n+1) x (mu+1) lattice F; corridor=(mn_lo, mn_hi) or None."""
    x = np.ascontiguousarray(x, dtype=np.uint8)
    y = np.ascontiguousarray(y, dtype=np.uint8)
    n, mu = len(x), len(y)
    F = np.zeros((n + 1, mu + 1), dtype=np.float64)
    lo, hi = corridor if corridor is not None else (0, 0)
    rc = _load().oracle_lattice(n, _ptr(x), mu, _ptr(y) if mu else None, Pi, Pd, Ps,
                                int(corridor is not None), lo, hi, _ptr(F))
    if rc != 0:
        raise ValueError("oracle_lattice: invalid arguments")
    return F


def receiver(x, y, Pi, Pd, Ps, corridor=None) -> float:
    """R(y|x) = F_{n,mu}."""
    return float(lattice(x, y, Pi, Pd, Ps, corridor)[-1, -1])


class Problem:
    """Decoder parameters shared by all frames (the decoder_create arguments)."""

    def __init__(self, q, n, N, C, Pi, Pd, Ps, mn, mt):
        self.q, self.n, self.N = int(q), int(n), int(N)
        self.C = np.ascontiguousarray(C, dtype=np.uint32).reshape(N, q)
        self.Pi, self.Pd, self.Ps = float(Pi), float(Pd), float(Ps)
        self.mn_lo, self.mn_hi = int(mn[0]), int(mn[1])
        self.mt_lo, self.mt_hi = int(mt[0]), int(mt[1])

    @property
    def Mt(self):
        return self.mt_hi - self.mt_lo + 1

    @property
    def Mn(self):
        return self.mn_hi - self.mn_lo + 1

    def _args(self):
        return (self.q, self.n, self.N, _ptr(self.C), self.Pi, self.Pd, self.Ps,
                self.mn_lo, self.mn_hi, self.mt_lo, self.mt_hi)


def gamma(prob: Problem, y, i: int, priors=None):
    """gamma_i(m', m, D) as array [M_tau][M_n][q] (eqn:gamma)."""
    y = np.ascontiguousarray(y, dtype=np.uint8)
    pr = None if priors is None else np.ascontiguousarray(priors, dtype=np.float64).reshape(prob.N, prob.q)
    g = np.zeros((prob.Mt, prob.Mn, prob.q), dtype=np.float64)
    rc = _load().oracle_gamma_at(*prob._args(), _ptr(y) if len(y) else None, len(y), _ptr(pr), int(i), _ptr(g))
    if rc != 0:
        raise ValueError("oracle_gamma_at: invalid arguments")
    return g


def set_threads(t: int) -> int:
    """Host threads used inside ONE frame decode (gamma's m' loop, L's D loop, beta's m' loop).
    The result is bit-identical for every thread count (the loops split keep the serial order of
    every sum); the default 1 leaves frame-level threading (decode_many) to the caller."""
    return _load().oracle_set_threads(int(t))


def decode(prob: Problem, y, priors=None, want_states=False, alpha0=None, betaN=None, extrinsic=False):
    """Decode one frame.  Returns dict(status, L[N][q], log_lambda[, alpha, beta, logA, logB][, E]).

    alpha0 / betaN: optional frame-boundary priors over the M_tau states;
    default point masses delta(0), delta(rho - tau).  Threads inside the frame: set_threads()."""
    y = np.ascontiguousarray(y, dtype=np.uint8)
    pr = None if priors is None else np.ascontiguousarray(priors, dtype=np.float64).reshape(prob.N, prob.q)
    a0 = None if alpha0 is None else np.ascontiguousarray(alpha0, dtype=np.float64).reshape(prob.Mt)
    bN = None if betaN is None else np.ascontiguousarray(betaN, dtype=np.float64).reshape(prob.Mt)
    L = np.zeros((prob.N, prob.q), dtype=np.float64)
    ll = ctypes.c_double(0.0)
    extra = {}
    if want_states:
        extra = dict(alpha=np.zeros((prob.N + 1, prob.Mt)), beta=np.zeros((prob.N + 1, prob.Mt)),
                     logA=np.zeros(prob.N + 1), logB=np.zeros(prob.N + 1))
    rc = _load().oracle_decode(*prob._args(), _ptr(y) if len(y) else None, len(y), _ptr(pr), _ptr(a0), _ptr(bN), _ptr(L),
                               ctypes.cast(ctypes.pointer(ll), ctypes.c_void_p),
                               _ptr(extra.get("alpha")), _ptr(extra.get("beta")),
                               _ptr(extra.get("logA")), _ptr(extra.get("logB")))
    if rc < 0:
        raise ValueError("oracle_decode: invalid arguments")
    out = dict(status=rc, L=L, log_lambda=ll.value)
    out.update(extra)
    if extrinsic:
        E = np.zeros_like(L)
        _load().oracle_extrinsic(prob.N, prob.q, _ptr(L), _ptr(pr), _ptr(E))
        out["E"] = E
    return out


def decode_many(prob: Problem, ys, priors_list=None, threads=None, **kw):
    """Decode many frames on host threads (ctypes drops the GIL during the C call)."""
    threads = threads or os.cpu_count() or 1
    priors_list = priors_list if priors_list is not None else [None] * len(ys)
    _load()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda a: decode(prob, a[0], a[1], **kw), zip(ys, priors_list)))
