"""ctypes binding of ``include/bsidmap.h`` (same names, argument marshalling only).

Loads the in-tree ``libbsidmap.so`` (built by ``make`` / ``__graft_entry__.build()``).
There is no fallback: if the library is missing this module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbsidmap.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "bsidmap.h")

def source_digest() -> str:
    """sha256 (first 16 hex digits) of the library's sources (csrc/*.cu, *.cuh and the header): ties
    a stored profile (profiles/ncu_summary.json) to the kernels it measured; a stale one is refused."""
    import hashlib
    csrc = os.path.join(_HERE, "csrc")
    h = hashlib.sha256()
    for f in sorted(os.listdir(csrc)) + [HEADER_PATH]:
        path = f if os.path.isabs(f) else os.path.join(csrc, f)
        if path.endswith((".cu", ".cuh", ".h")):
            h.update(os.path.basename(path).encode())
            with open(path, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


BSIDMAP_OK = 0
BSIDMAP_EINVAL = -1
BSIDMAP_ENOTINJECTIVE = -2
BSIDMAP_ENOMEM = -3
BSIDMAP_EPLAN = -4
BSIDMAP_ECUDA = -5
BSIDMAP_FRAME_OK = 0
BSIDMAP_FRAME_DRIFT_OUT_OF_RANGE = 1
BSIDMAP_FRAME_UNDERFLOW = 2
BSIDMAP_MODE_AUTO = 0
BSIDMAP_MODE_STORED = 1
BSIDMAP_MODE_RECOMPUTE = 2
BSIDMAP_MODE_GAMMASUM = 3

_p, _i, _d, _sz, _l, _ll = (ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t,
                            ctypes.c_long, ctypes.c_longlong)

# name -> (restype, argtypes); mirrors include/bsidmap.h one to one
SIGNATURES = {
    "bsidmap_create": (_i, [ctypes.POINTER(_p), _i, _i, _i, _p, _d, _d, _d, _i, _i, _i, _i, _i, _i]),
    "bsidmap_decode_batch": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _p]),
    "bsidmap_decode_batch_host": (_i, [_p, _i, _p, _sz, _p, _p, _p, _p, _p, _p]),
    "bsidmap_decode_batch_opts": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _p, _p]),
    "bsidmap_destroy": (None, [_p]),
    "bsidmap_last_error": (ctypes.c_char_p, [_p]),
    "bsidmap_workspace_bytes": (_sz, [_p, _i, _i]),
    "bsidmap_set_workspace_limit": (_i, [_p, _sz]),
    "bsidmap_set_mode": (_i, [_p, _i]),
    "bsidmap_set_timing": (_i, [_p, _i]),
    "bsidmap_phase_times": (_i, [_p, _p, _i]),
    "bsidmap_last_launch_count": (_l, [_p]),
    "bsidmap_plan_info": (_i, [_p, _i, ctypes.c_char_p, _sz]),
    "bsidmap_lattice_nodes": (_l, [_p]),
    "bsidmap_valid_lattices": (_ll, [_p, _i, _p]),
    "bsidmap_debug_gamma": (_i, [_p, _i, _p, _p, _p, _p, _i, _p, _p]),
    "bsidmap_debug_states": (_i, [_p, _i, _p, _p, _p]),
    "bsidmap_drift_pmf": (_i, [_i, _d, _d, _i, _i, _p]),
    "bsidmap_drift_limits": (_i, [_i, _d, _d, _d, _p, _p]),
    "bsidmap_drift_limits_tails": (_i, [_i, _d, _d, _d, _p, _p]),
    "bsidmap_jit_compile": (_i, [_i, _i, _i, ctypes.c_char_p, _sz]),
    "bsidmap_state_space": (_i, [_i, _i, _d, _d, _d, _p, _p, _p, _p]),
    "bsidmap_phi": (_i, [_i, _d, _d, _i, _i, _i, _p, _p]),
    "bsidmap_mc_generate": (_i, [_p, ctypes.c_uint64, ctypes.c_int64, _i, _i, _p, _p, _p, _p, _p]),
    "bsidmap_count_errors": (_i, [_p, _i, _p, _p, _p, _p, _p]),
    "bsidmap_mc_run": (_i, [_p, ctypes.c_uint64, ctypes.c_int64, _i, _i, _p, _p]),
}

_lib = None


def load():
    """Load libbsidmap.so (raises OSError if it was not built -- no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build() (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class DecodeOpts(ctypes.Structure):
    """struct bsidmap_decode_opts (device pointers)."""
    _fields_ = [("alpha0", ctypes.c_void_p), ("betaN", ctypes.c_void_p), ("extrinsic", ctypes.c_void_p)]


class BsidmapError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"bsidmap error {code}: {msg}")
        self.code = code


def check(rc, handle=None):
    if rc != BSIDMAP_OK:
        msg = load().bsidmap_last_error(handle)
        raise BsidmapError(rc, msg.decode() if msg else "")
    return rc
