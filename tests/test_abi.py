"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/*.h declares, the binding covers them, and bsidmap_create rejects bad
arguments before touching the device."""
import ctypes
import glob
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1802_08483_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(bsidmap_[a-z_]+)\s*\(", src))
    return names


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("bsidmap_create", "bsidmap_decode_batch", "bsidmap_destroy", "bsidmap_last_error",
                 "bsidmap_decode_batch_host", "bsidmap_workspace_bytes"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_lib.SIGNATURES) == _declared()


def test_library_is_sm100a_native():
    """The shared object carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(**kw):
    args = dict(q=4, n=3, N=2, C=np.array([[0, 1, 2, 3], [4, 5, 6, 7]], np.uint32), Pi=0.01, Pd=0.01, Ps=0.0,
                mn=(-1, 1), mt=(-2, 2), mode=0)
    args.update(kw)
    h = ctypes.c_void_p()
    C = np.ascontiguousarray(args["C"], dtype=np.uint32)
    rc = _lib.load().bsidmap_create(ctypes.byref(h), args["q"], args["n"], args["N"],
                                    C.ctypes.data_as(ctypes.c_void_p), args["Pi"], args["Pd"], args["Ps"],
                                    args["mn"][0], args["mn"][1], args["mt"][0], args["mt"][1], args["mode"], 0)
    return rc, h


@pytest.mark.parametrize("kw,code", [
    (dict(q=1), _lib.BSIDMAP_EINVAL),
    (dict(q=16), _lib.BSIDMAP_EINVAL),                       # q > 2^n
    (dict(n=0), _lib.BSIDMAP_EINVAL),
    (dict(Pi=0.6, Pd=0.5), _lib.BSIDMAP_EINVAL),             # Pi + Pd >= 1
    (dict(Ps=1.5), _lib.BSIDMAP_EINVAL),
    (dict(mn=(1, 2)), _lib.BSIDMAP_EINVAL),                  # corridor must contain 0
    (dict(mt=(0, 2)), _lib.BSIDMAP_EINVAL),                  # m_tau^- > m_n^-
    (dict(mn=(-20, 20), mt=(-20, 20)), _lib.BSIDMAP_EPLAN),  # M_n = 41 > 32
    (dict(C=np.array([[0, 1, 2, 2], [4, 5, 6, 7]])), _lib.BSIDMAP_ENOTINJECTIVE),
    (dict(C=np.array([[0, 1, 2, 8], [4, 5, 6, 7]])), _lib.BSIDMAP_EINVAL),  # bit above n
    (dict(mode=7), _lib.BSIDMAP_EINVAL),
])
def test_create_rejects_bad_arguments(kw, code):
    rc, h = _create(**kw)
    assert rc == code
    assert not h.value
    assert _lib.load().bsidmap_last_error(None)


def test_null_decoder_calls_fail_cleanly():
    lib = _lib.load()
    assert lib.bsidmap_decode_batch(None, 1, None, None, None, None, None, None, None) == _lib.BSIDMAP_EINVAL
    assert lib.bsidmap_workspace_bytes(None, 10, 0) == 0
    lib.bsidmap_destroy(None)


def test_c_example_builds_and_links():
    """The C ABI is usable from plain C: examples/decode_host.c compiles against include/bsidmap.h
    and links against the library (run on the GPU box by test_gpu_edges.test_c_example_runs)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "decode_host")
    r = subprocess.run(["make", "-C", root, "examples/decode_host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert os.path.exists(exe)


def test_jit_compiles_a_shape_without_a_unit(tmp_path, monkeypatch):
    """NVRTC compiles the unrolled kernels of a shape with no compiled unit (J1's corridor) for
    sm_100a without a device, into five cached programs; shapes beyond the unrolled cores' bounds
    are refused with a reason (the decoder then keeps the generic core)."""
    monkeypatch.setenv("BSIDMAP_JIT_CACHE", str(tmp_path))
    lib = _lib.load()
    buf = ctypes.create_string_buffer(4096)
    assert lib.bsidmap_jit_compile(9, -7, 17, buf, 4096) == _lib.BSIDMAP_OK, buf.value
    assert len(list(tmp_path.iterdir())) == 5
    assert lib.bsidmap_jit_compile(40, -1, 24, buf, 4096) == _lib.BSIDMAP_EPLAN
    assert b"corridor nodes" in buf.value
