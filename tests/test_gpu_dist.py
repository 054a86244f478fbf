"""The multi-rank path of bench.py decoding for real: two ranks share the one B200 of the test box
(torchrun, BSIDMAP_DIST_BACKEND=gloo for the reductions), each decodes its own contiguous shard of
the global frames (frames are independent, no data-path collective), and every rank's
L and status must equal -- bit for bit -- the single-process decode of the same global frames.
The job-wide counts in the bench line (frames, frames_ok, symbol errors) are sums over ranks.
Frame sharding is this build's own axis; the paper's decoder is single-GPU."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import bsidgen

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("config,N,shard", [
    ("C2", None, ["--frames", "96"]),                       # weak scaling: 96 frames per rank
    ("C5", 60, ["--frames", "5"]),                          # C5's code/channel/trellis, N cut to 60
    ("C5", None, ["--total-frames", "256", "--ws-limit-gb", "40"]),  # full C5, strong: 128 per rank, chunked
])
def test_two_ranks_equal_single_process(config, N, shard, tmp_path):
    world = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--config", config, "--steps", "1", "--warmup", "1", "--no-cpu-baseline",
           "--no-e2e", "--dump", str(tmp_path)] + shard + ([] if N is None else ["--N", str(N)])
    env = dict(os.environ, BSIDMAP_DIST_BACKEND="gloo")
    p = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == world

    import dataclasses
    cfg = bsidgen.configs()[config]
    if N is not None:
        cfg = dataclasses.replace(cfg, N=N)
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    firsts = [int(x["first"]) for x in parts]
    counts = [int(x["count"]) for x in parts]
    assert firsts[0] == 0 and firsts[1] == counts[0]
    total = sum(counts)
    assert line["config"]["total_frames"] == total

    from paper_1802_08483_b200 import Decoder
    b = bsidgen.make_batch(cfg, 0, total)
    d = Decoder.from_config(cfg, b.C, device=0)
    dev = torch.device("cuda", 0)
    pri = torch.from_numpy(b.priors).to(dev) if b.priors is not None else None
    L, st = d.decode(torch.from_numpy(b.rx.ravel().copy()).to(dev), torch.from_numpy(b.offsets).to(dev),
                     torch.from_numpy(b.rho).to(dev), pri)
    torch.cuda.synchronize()
    L, st = L.cpu().numpy(), st.cpu().numpy()
    for x, f0, c in zip(parts, firsts, counts):
        np.testing.assert_array_equal(x["status"], st[f0:f0 + c])
        np.testing.assert_array_equal(x["L"], L[f0:f0 + c])
    # job-wide counts are sums over the ranks' shards
    assert line["frames_ok"] == pytest.approx((st == 0).mean())
    ser = (np.argmax(L, 2) != b.msg).sum() / (total * cfg.N)
    assert line["symbol_error_rate"] == pytest.approx(ser, rel=1e-12, abs=1e-15)
