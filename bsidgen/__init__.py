"""Seeded synthetic workloads for the BSID MAP decoder (arXiv 1802.08483).

Shared by the oracle tests, the CUDA parity tests and ``bench.py``.  This
module holds none of the decoder's arithmetic: it draws codebooks, messages,
BSID channel outputs and priors (``bsidgen.c``), packs/unpacks bits, and
sizes the drift state space with the harness rule of DESIGN.md reading R8
(exact drift PMF, exclusion probability P_r = 1e-10; the paper defers this
rule to bbw14joe).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bsidgen.c")
_LIB_PATH = os.path.join(_HERE, "libbsidgen.so")
_lock = threading.Lock()
_lib = None

MASTER_SEED = 1802_08483


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            p, i, d, u64, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_int64
            lib.gen_codebook.restype = i
            lib.gen_codebook.argtypes = [u64, i, i, i, p]
            lib.gen_frames.restype = i64
            lib.gen_frames.argtypes = [u64, i64, i, i, i, i, p, d, d, d, i, i, i, p, p, p]
            lib.gen_priors.restype = i
            lib.gen_priors.argtypes = [u64, i64, i, i, i, p, p]
            _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# drift PMF and state-space limits (harness rule, reading R8)
# ---------------------------------------------------------------------------

def bit_drift_pmf(Pi: float, Pd: float, tail: float = 1e-17, kmax: int = 64):
    """PMF of the drift change over one transmitted bit.

    k insertions then deletion: change k-1 w.p. Pi^k Pd; k insertions then
    transmission: change k w.p. Pi^k Pt.  Returns (offset, pmf) with
    pmf[j] = P(change = offset + j), offset = -1.
    """
    Pt = 1.0 - Pi - Pd
    K = 0
    while K < kmax and Pi > 0 and Pi ** (K + 1) >= tail:
        K += 1
    pmf = np.zeros(K + 2)
    for k in range(K + 1):
        pmf[k - 1 + 1] += Pi ** k * Pd
        pmf[k + 1] += Pi ** k * Pt
    return -1, pmf


def drift_pmf(T: int, Pi: float, Pd: float, floor: float = 1e-300):
    """Exact PMF of the drift S_T after T bits: T-fold convolution by squaring.

    Returns (offset, pmf) with pmf[j] = P(S_T = offset + j).
    """
    off1, p1 = bit_drift_pmf(Pi, Pd)
    res_off, res = 0, np.array([1.0])
    base_off, base = off1, p1
    t = int(T)
    while t > 0:
        if t & 1:
            res = np.convolve(res, base)
            res_off += base_off
            res, res_off = _trim(res, res_off, floor)
        t >>= 1
        if t:
            base = np.convolve(base, base)
            base_off *= 2
            base, base_off = _trim(base, base_off, floor)
    return res_off, res


def _trim(p, off, floor):
    nz = np.nonzero(p > floor)[0]
    if len(nz) == 0:
        return p, off
    return p[nz[0]:nz[-1] + 1].copy(), off + int(nz[0])


def drift_limits(T: int, Pi: float, Pd: float, Pr: float = 1e-10, rule: str = "greedy"):
    """(m_T^-, m_T^+) with exclusion probability Pr (reading R8).

    rule "greedy" (default): grow [0, 0] one state at a time on the side with more
    excluded mass (ties: the positive side) until P(S_T < m^-) + P(S_T > m^+) < Pr.
    rule "tails" (round 1): m^- = max{m : P(S_T < m) <= Pr/2}, m^+ = min{m : P(S_T > m) <= Pr/2},
    clamped to -T <= m^- <= 0 <= m^+.
    """
    off, p = drift_pmf(T, Pi, Pd)
    if rule == "greedy":
        mass = float(p.sum())
        if not (1.0 - mass < Pr):
            raise ValueError("drift PMF truncation loss >= Pr")
        left = np.concatenate([[0.0], np.cumsum(p)])              # left[j] = P(S < off + j)
        right = np.concatenate([np.cumsum(p[::-1])[::-1][1:], [0.0]])  # right[j] = P(S > off + j)

        def below(m):
            j = m - off
            return 0.0 if j <= 0 else mass if j >= len(p) else float(left[j])

        def above(m):
            j = m - off
            return 0.0 if j >= len(p) else mass if j < 0 else float(right[j])

        lo = hi = 0
        while below(lo) + above(hi) >= Pr:
            if above(hi) >= below(lo):
                hi += 1
            else:
                lo -= 1
        return int(lo), int(hi)
    assert rule == "tails", rule
    cdf = np.cumsum(p)             # cdf[j] = P(S <= off + j)
    lo = 0
    for j in range(len(p)):        # P(S < off + j) = cdf[j-1]
        below = cdf[j - 1] if j > 0 else 0.0
        if below <= Pr / 2:
            lo = off + j
        else:
            break
    sf = np.cumsum(p[::-1])[::-1]  # sf[j] = P(S >= off + j)
    hi = off + len(p) - 1
    for j in range(len(p) - 1, -1, -1):  # P(S > off + j) = sf[j+1]
        above = sf[j + 1] if j + 1 < len(p) else 0.0
        if above <= Pr / 2:
            hi = off + j
        else:
            break
    lo = max(min(lo, 0), -T)
    hi = max(hi, 0)
    return int(lo), int(hi)


# ---------------------------------------------------------------------------
# configurations (BASELINE.json "configs", SURVEY 8 sizing table)
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class Config:
    name: str
    q: int
    n: int
    N: int
    Pi: float
    Pd: float
    Ps: float
    frames: int
    priors: bool = False
    mn: tuple | None = None
    mt: tuple | None = None
    seed: int = MASTER_SEED

    def __post_init__(self):
        if self.mn is None:
            self.mn = drift_limits(self.n, self.Pi, self.Pd)
        if self.mt is None:
            lo, hi = drift_limits(self.tau, self.Pi, self.Pd)
            self.mt = (min(lo, self.mn[0]), max(hi, self.mn[1]))

    @property
    def tau(self):
        return self.n * self.N

    @property
    def Mn(self):
        return self.mn[1] - self.mn[0] + 1

    @property
    def Mt(self):
        return self.mt[1] - self.mt[0] + 1

    @property
    def words_per_frame(self):
        return (self.tau + self.mt[1] + 31) // 32 + 1

    def to_dict(self):
        return dict(name=self.name, q=self.q, n=self.n, N=self.N, Pi=self.Pi, Pd=self.Pd, Ps=self.Ps,
                    frames=self.frames, priors=self.priors, mn=list(self.mn), mt=list(self.mt))


def configs():
    """C1..C5 of BASELINE.json (Ps=0 where unspecified: the paper's setting)."""
    return {
        "C1": Config("C1", q=8, n=7, N=10, Pi=0.01, Pd=0.01, Ps=0.0, frames=1, seed=MASTER_SEED + 1),
        "C2": Config("C2", q=16, n=10, N=100, Pi=0.01, Pd=0.01, Ps=0.001, frames=65536, seed=MASTER_SEED + 2),
        "C3": Config("C3", q=32, n=8, N=500, Pi=0.05, Pd=0.05, Ps=0.0, frames=16384, seed=MASTER_SEED + 3),
        "C4": Config("C4", q=16, n=10, N=1000, Pi=0.1, Pd=0.1, Ps=0.0, frames=4096, seed=MASTER_SEED + 4),
        "C5": Config("C5", q=64, n=12, N=10000, Pi=0.02, Pd=0.02, Ps=0.0, frames=256, priors=True,
                     seed=MASTER_SEED + 5),
    }


def extra_configs():
    """Shapes outside BASELINE.json (no compiled unit: the decoder compiles their unrolled core at
    create, jit.cu).  J1: a q = 32, n = 9 code on a Pi = Pd = 0.03 channel, the C2 batch size."""
    return {
        "J1": Config("J1", q=32, n=9, N=100, Pi=0.03, Pd=0.03, Ps=0.0, frames=65536, seed=MASTER_SEED + 11),
    }


def all_configs():
    return {**configs(), **extra_configs()}


@dataclasses.dataclass
class Batch:
    cfg: Config
    first: int
    C: np.ndarray        # [N][q] uint32
    msg: np.ndarray      # [F][N] int32
    rx: np.ndarray       # [F][words_per_frame] uint32, LSB-first
    rho: np.ndarray      # [F] int32
    offsets: np.ndarray  # [F] int64 word offsets into rx.ravel()
    priors: np.ndarray | None  # [F][N][q] float32
    redraws: int

    def bits(self, f: int) -> np.ndarray:
        """Unpacked received bits of frame f (uint8, y_1 first)."""
        return unpack_bits(self.rx[f], int(self.rho[f]))


def codebook(cfg: Config) -> np.ndarray:
    C = np.zeros((cfg.N, cfg.q), dtype=np.uint32)
    if _load().gen_codebook(cfg.seed, cfg.N, cfg.q, cfg.n, _ptr(C)) != 0:
        raise ValueError("gen_codebook: bad arguments")
    return C


def make_batch(cfg: Config, first: int = 0, count: int | None = None, C: np.ndarray | None = None) -> Batch:
    """Frames [first, first+count) of cfg's seeded workload."""
    count = cfg.frames if count is None else int(count)
    C = codebook(cfg) if C is None else C
    wpf = cfg.words_per_frame
    msg = np.zeros((count, cfg.N), dtype=np.int32)
    rx = np.zeros((count, wpf), dtype=np.uint32)
    rho = np.zeros(count, dtype=np.int32)
    red = _load().gen_frames(cfg.seed, int(first), count, cfg.N, cfg.q, cfg.n, _ptr(C), cfg.Pi, cfg.Pd, cfg.Ps,
                             cfg.mt[0], cfg.mt[1], wpf, _ptr(msg), _ptr(rx), _ptr(rho))
    if red < 0:
        raise ValueError("gen_frames: bad arguments")
    pri = None
    if cfg.priors:
        pri = np.zeros((count, cfg.N, cfg.q), dtype=np.float32)
        if _load().gen_priors(cfg.seed, int(first), count, cfg.N, cfg.q, _ptr(msg), _ptr(pri)) != 0:
            raise ValueError("gen_priors: bad arguments")
    offsets = np.arange(count, dtype=np.int64) * wpf
    return Batch(cfg, int(first), C, msg, rx, rho, offsets, pri, int(red))


def unpack_bits(words: np.ndarray, nbits: int) -> np.ndarray:
    b = np.unpackbits(np.ascontiguousarray(words, dtype="<u4").view(np.uint8), bitorder="little")
    return b[:nbits].astype(np.uint8)


def pack_bits(bits, words: int | None = None) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint8)
    nw = (len(bits) + 31) // 32 if words is None else words
    buf = np.zeros(nw * 32, dtype=np.uint8)
    buf[:len(bits)] = bits
    return np.packbits(buf, bitorder="little").view("<u4").astype(np.uint32)


def encode(C: np.ndarray, msg, n: int) -> np.ndarray:
    """X = C_0(D_0) || ... || C_{N-1}(D_{N-1}) as bits."""
    out = []
    for i, D in enumerate(msg):
        w = int(C[i, D])
        out.extend((w >> t) & 1 for t in range(n))
    return np.array(out, dtype=np.uint8)
