"""Thin Python face of the C ABI: a ``Decoder`` owning one ``bsidmap_decoder``.

Every method is argument marshalling around one ``bsidmap_*`` call; all
decoding runs in the CUDA kernels of ``libbsidmap.so``.
"""
from __future__ import annotations

import ctypes
import json

import numpy as np
import torch

from . import _lib


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Decoder:
    """bsidmap_create / bsidmap_destroy for one device."""

    def __init__(self, q, n, N, codebook, Pi, Pd, Ps, mn, mt, mode=_lib.BSIDMAP_MODE_AUTO, device=None):
        self._lib = _lib.load()
        C = np.ascontiguousarray(codebook, dtype=np.uint32).reshape(N, q)
        dev = torch.cuda.current_device() if device is None else int(device)
        h = ctypes.c_void_p()
        rc = self._lib.bsidmap_create(ctypes.byref(h), q, n, N, C.ctypes.data_as(ctypes.c_void_p),
                                      float(Pi), float(Pd), float(Ps), int(mn[0]), int(mn[1]),
                                      int(mt[0]), int(mt[1]), int(mode), dev)
        _lib.check(rc, None)
        self.h = h
        self.q, self.n, self.N = q, n, N
        self.mn, self.mt = tuple(mn), tuple(mt)
        self.device = torch.device("cuda", dev)

    @classmethod
    def from_config(cls, cfg, C, mode=_lib.BSIDMAP_MODE_AUTO, device=None):
        return cls(cfg.q, cfg.n, cfg.N, C, cfg.Pi, cfg.Pd, cfg.Ps, cfg.mn, cfg.mt, mode, device)

    def close(self):
        if getattr(self, "h", None):
            self._lib.bsidmap_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ decode
    def decode_batch(self, rx, rx_off, rho, priors, L, status, stream=None):
        """bsidmap_decode_batch on device tensors (async on `stream`)."""
        F = int(rho.numel())
        rc = self._lib.bsidmap_decode_batch(self.h, F, _ptr(rx), _ptr(rx_off), _ptr(rho), _ptr(priors),
                                            _ptr(L), _ptr(status), _stream(stream))
        _lib.check(rc, self.h)

    def decode(self, rx, rx_off, rho, priors=None, stream=None, alpha0=None, betaN=None, extrinsic=False):
        """Allocate outputs and decode; returns (L [F][N][q] fp32, status [F] int32) on the device,
        plus E (extrinsic) if requested.  alpha0/betaN: [F][M_tau] fp64 boundary priors."""
        F = int(rho.numel())
        L = torch.empty((F, self.N, self.q), dtype=torch.float32, device=self.device)
        st = torch.empty((F,), dtype=torch.int32, device=self.device)
        if alpha0 is None and betaN is None and not extrinsic:
            self.decode_batch(rx, rx_off, rho, priors, L, st, stream)
            return L, st
        E = torch.empty_like(L) if extrinsic else None
        opts = _lib.DecodeOpts(None if alpha0 is None else alpha0.data_ptr(),
                               None if betaN is None else betaN.data_ptr(), None if E is None else E.data_ptr())
        rc = self._lib.bsidmap_decode_batch_opts(self.h, F, _ptr(rx), _ptr(rx_off), _ptr(rho), _ptr(priors),
                                                 ctypes.byref(opts), _ptr(L), _ptr(st), _stream(stream))
        _lib.check(rc, self.h)
        return (L, st, E) if extrinsic else (L, st)

    def decode_host(self, rx, rx_off, rho, priors, L, status, stream=None):
        """bsidmap_decode_batch_host on host (ideally pinned) tensors/arrays; synchronous."""
        F = int(len(rho))
        nw = int(rx.numel() if isinstance(rx, torch.Tensor) else rx.size)
        rc = self._lib.bsidmap_decode_batch_host(self.h, F, _ptr(rx), nw, _ptr(rx_off), _ptr(rho), _ptr(priors),
                                                 _ptr(L), _ptr(status), _stream(stream))
        _lib.check(rc, self.h)

    # --------------------------------------------------------------- planning
    def workspace_bytes(self, F, mode=_lib.BSIDMAP_MODE_AUTO):
        return int(self._lib.bsidmap_workspace_bytes(self.h, int(F), int(mode)))

    def set_workspace_limit(self, nbytes):
        _lib.check(self._lib.bsidmap_set_workspace_limit(self.h, int(nbytes)), self.h)

    def set_mode(self, mode):
        _lib.check(self._lib.bsidmap_set_mode(self.h, int(mode)), self.h)

    def plan(self, F):
        buf = ctypes.create_string_buffer(2048)
        rc = self._lib.bsidmap_plan_info(self.h, int(F), buf, 2048)
        if rc < 0:
            _lib.check(rc, self.h)
        return json.loads(buf.value.decode())

    def set_timing(self, on=True):
        _lib.check(self._lib.bsidmap_set_timing(self.h, int(bool(on))), self.h)

    def phase_times(self):
        arr = (ctypes.c_float * 8)()
        k = self._lib.bsidmap_phase_times(self.h, arr, 8)
        if k < 0:
            _lib.check(k, self.h)
        return list(arr)[:k]

    def last_launch_count(self):
        return int(self._lib.bsidmap_last_launch_count(self.h))

    def lattice_nodes(self):
        return int(self._lib.bsidmap_lattice_nodes(self.h))

    def valid_lattices(self, rho_host):
        r = np.ascontiguousarray(rho_host, dtype=np.int32)
        return int(self._lib.bsidmap_valid_lattices(self.h, len(r), r.ctypes.data_as(ctypes.c_void_p)))

    # ------------------------------------------------------------- Monte Carlo
    def mc_generate(self, seed, first, F, words_per_frame, stream=None):
        """Device-generated frames (bsidmap_mc_generate): (msg, rx, rho, redraws) tensors."""
        msg = torch.empty((F, self.N), dtype=torch.int32, device=self.device)
        rx = torch.zeros((F, words_per_frame), dtype=torch.int32, device=self.device)
        rho = torch.empty((F,), dtype=torch.int32, device=self.device)
        red = torch.zeros((1,), dtype=torch.int64, device=self.device)
        _lib.check(self._lib.bsidmap_mc_generate(self.h, int(seed), int(first), int(F), int(words_per_frame), _ptr(msg),
                                                 _ptr(rx), _ptr(rho), _ptr(red), _stream(stream)), self.h)
        return msg, rx, rho, red

    def count_errors(self, L, msg, status, counters=None, stream=None):
        """bsidmap_count_errors; returns the device counters [symbol errors, frame errors, failed]."""
        counters = torch.zeros((3,), dtype=torch.int64, device=self.device) if counters is None else counters
        _lib.check(self._lib.bsidmap_count_errors(self.h, int(msg.shape[0]), _ptr(L), _ptr(msg), _ptr(status),
                                                  _ptr(counters), _stream(stream)), self.h)
        return counters

    def mc_run(self, seed, first, F, batch, stream=None):
        """bsidmap_mc_run: dict(frames, symbol_errors, frame_errors, redraws)."""
        res = (ctypes.c_ulonglong * 4)()
        _lib.check(self._lib.bsidmap_mc_run(self.h, int(seed), int(first), int(F), int(batch), res, _stream(stream)),
                   self.h)
        return dict(frames=res[0], symbol_errors=res[1], frame_errors=res[2], redraws=res[3])

    # ------------------------------------------------------------------ debug
    def debug_gamma(self, rx, rx_off, rho, priors, i, stream=None):
        F = int(rho.numel())
        Mt, Mn = self.mt[1] - self.mt[0] + 1, self.mn[1] - self.mn[0] + 1
        out = torch.empty((F, Mt, Mn, self.q), dtype=torch.float64, device=self.device)
        rc = self._lib.bsidmap_debug_gamma(self.h, F, _ptr(rx), _ptr(rx_off), _ptr(rho), _ptr(priors), int(i),
                                           _ptr(out), _stream(stream))
        _lib.check(rc, self.h)
        return out

    def debug_states(self, F, stream=None):
        Mt = self.mt[1] - self.mt[0] + 1
        a = torch.empty((F, self.N + 1, Mt), dtype=torch.float64, device=self.device)
        b = torch.empty_like(a)
        _lib.check(self._lib.bsidmap_debug_states(self.h, int(F), _ptr(a), _ptr(b), _stream(stream)), self.h)
        return a, b


# ---------------------------------------------------------------- state-space sizing (host)
def drift_pmf(T, Pi, Pd, lo, hi):
    """P(S_T = m) for m in [lo, hi] (bsidmap_drift_pmf)."""
    lib = _lib.load()
    out = np.zeros(hi - lo + 1, dtype=np.float64)
    _lib.check(lib.bsidmap_drift_pmf(int(T), float(Pi), float(Pd), int(lo), int(hi), _ptr(out)))
    return out


def drift_limits(T, Pi, Pd, Pr=1e-10, rule="greedy"):
    """(m_T^-, m_T^+) with exclusion probability Pr: rule "greedy" = bsidmap_drift_limits (smallest
    interval around 0, total excluded mass < Pr), "tails" = bsidmap_drift_limits_tails."""
    lib = _lib.load()
    lo, hi = ctypes.c_int(), ctypes.c_int()
    fn = {"greedy": lib.bsidmap_drift_limits, "tails": lib.bsidmap_drift_limits_tails}[rule]
    _lib.check(fn(int(T), float(Pi), float(Pd), float(Pr), ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def state_space(n, N, Pi, Pd, Pr=1e-10):
    """((m_n^-, m_n^+), (m_tau^-, m_tau^+)) (bsidmap_state_space)."""
    lib = _lib.load()
    v = [ctypes.c_int() for _ in range(4)]
    _lib.check(lib.bsidmap_state_space(int(n), int(N), float(Pi), float(Pd), float(Pr), *[ctypes.byref(x) for x in v]))
    return (v[0].value, v[1].value), (v[2].value, v[3].value)


def phi(T, Pi, Pd, lo, hi, num_frames, device=None, stream=None):
    """Phi_T on the device: [num_frames][hi - lo + 1] drift PMF (bsidmap_phi)."""
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty((num_frames, hi - lo + 1), dtype=torch.float64, device=dev)
    _lib.check(lib.bsidmap_phi(int(T), float(Pi), float(Pd), int(lo), int(hi), int(num_frames), _ptr(out),
                               _stream(stream)))
    return out
