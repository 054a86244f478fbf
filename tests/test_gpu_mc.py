"""NEXT-3: the Monte-Carlo SER/FER workload on the device.
The device generator must reproduce the host generator bit for bit (same counter-based
stream, the literal BSID event loop), and the error counts must equal a host
count of the same decoder outputs."""
import numpy as np
import pytest
import torch

import bsidgen
from tests.test_gpu_parity import _dec, small_cfg, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,over", [("C1", {}), ("C2", {}), ("C4", {}), ("C2", {"mn": (-2, 2), "mt": (-3, 3)})])
def test_device_generator_equals_host(name, over):
    cfg = small_cfg(name, **over)
    F = 64 if name != "C4" else 8
    b = bsidgen.make_batch(cfg, 1000, F)
    d = _dec().from_config(cfg, b.C, device=0)
    msg, rx, rho, red = d.mc_generate(cfg.seed, 1000, F, cfg.words_per_frame)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(msg.cpu().numpy(), b.msg)
    np.testing.assert_array_equal(rho.cpu().numpy(), b.rho)
    np.testing.assert_array_equal(rx.cpu().numpy().view(np.uint32), b.rx)
    assert int(red.item()) == b.redraws
    if "mt" in over:
        assert b.redraws > 0  # the narrow state space forces redraws


def test_count_errors_and_mc_run_match_host():
    cfg = small_cfg("C2")
    F = 2000
    b = bsidgen.make_batch(cfg, 0, F)
    d = _dec().from_config(cfg, b.C, device=0)
    rx, off, rho, pri = to_dev(b)
    L, st = d.decode(rx, off, rho, pri)
    msg = torch.from_numpy(b.msg).to(L.device)
    cnt = d.count_errors(L, msg, st).cpu().numpy()
    Lh, sth = L.cpu().numpy(), st.cpu().numpy()
    dec = np.argmax(Lh, 2)
    wrong = (dec != b.msg) | (sth != 0)[:, None]
    assert cnt[0] == wrong.sum() and cnt[1] == wrong.any(1).sum() and cnt[2] == (sth != 0).sum()
    # the fused device loop (generate -> decode -> count) over two batches gives the same counts
    res = d.mc_run(cfg.seed, 0, F, 1000)
    assert res["frames"] == F and res["symbol_errors"] == cnt[0] and res["frame_errors"] == cnt[1]
    assert res["redraws"] == b.redraws
    assert 0.0 < cnt[0] / (F * cfg.N) < 0.1
