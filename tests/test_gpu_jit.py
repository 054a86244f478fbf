"""Run-time compiled lattice cores (jit.cu): a shape without a compiled unit gets the fully unrolled
kernels of the inst_spec_* units, compiled with NVRTC at bsidmap_create (the paper's templates over
the code and channel sizes, for any shape).  Parity against the FP64 oracle at the
north-star gate, and agreement with the generic core the same shape ran on before."""
import numpy as np
import pytest

import bsidgen
from .test_gpu_parity import _dec, assert_parity, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def _j1(N=20):
    import dataclasses
    return dataclasses.replace(bsidgen.extra_configs()["J1"], N=N)


@pytest.mark.parametrize("mode", [3, 2, 1])
def test_jit_shape_parity(mode, monkeypatch):
    cfg = _j1()
    b = bsidgen.make_batch(cfg, 3, 6)
    d, L, st = run_gpu(cfg, b, mode)
    pl = d.plan(6)
    assert pl["core"] == "jit", pl
    res = run_oracle(cfg, b)
    assert_parity(L, st, res)
    monkeypatch.setenv("BSIDMAP_JIT", "0")
    dg, Lg, stg = run_gpu(cfg, b, mode)
    assert dg.plan(6)["core"] == "generic"
    np.testing.assert_array_equal(st, stg)
    assert_parity(Lg, stg, res)


@pytest.mark.parametrize("k", range(4))
def test_jit_random_shapes(k):
    """Random codes and channels whose corridor has no compiled unit (pair and scalar APP cores,
    with and without priors), all three schedules."""
    rng = np.random.default_rng(100 + k)
    n = int(rng.integers(5, 12))
    q = int(rng.integers(3, min(64, 1 << n)))
    p = float(rng.choice([0.01, 0.03, 0.06]))
    cfg = bsidgen.Config(f"JR{k}", q=q, n=n, N=int(rng.integers(3, 25)), Pi=p, Pd=p, Ps=float(rng.choice([0.0, 0.01])),
                         frames=0, priors=bool(k % 2), seed=500 + k)
    b = bsidgen.make_batch(cfg, 0, int(rng.integers(2, 12)))
    res = run_oracle(cfg, b)
    for mode in (1, 2, 3):
        d, L, st = run_gpu(cfg, b, mode)
        assert d.plan(2)["core"] in ("jit", "spec"), d.plan(2)
        assert_parity(L, st, res)


def test_jit_cache_reuse(tmp_path, monkeypatch):
    """A shape compiled once is read back from the disk cache (and, within a process, from the
    loaded table): the second create of the same shape is fast."""
    import time
    monkeypatch.setenv("BSIDMAP_JIT_CACHE", str(tmp_path))
    cfg = bsidgen.Config("JC", q=12, n=8, N=5, Pi=0.02, Pd=0.02, Ps=0.0, frames=0, seed=41)
    C = bsidgen.codebook(cfg)
    t0 = time.time()
    d = _dec().from_config(cfg, C, device=0)
    t1 = time.time()
    assert d.plan(4)["core"] == "jit"
    assert len(list(tmp_path.iterdir())) == 5
    d2 = _dec().from_config(cfg, C, device=0)
    t2 = time.time()
    assert d2.plan(4)["core"] == "jit"
    assert t2 - t1 < max(1.0, 0.2 * (t1 - t0))
