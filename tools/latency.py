"""Single-frame decode latency (C1, the paper's small worked configuration): eager
bsidmap_decode_batch vs a CUDA-graph replay of the same call, device time per decode over
1000 back-to-back decodes (CUDA events on the stream)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bsidgen  # noqa: E402
from paper_1802_08483_b200 import Decoder  # noqa: E402

res = {}
for name, F in (("C1", 1), ("C1", 64), ("C2", 1)):
    cfg = bsidgen.configs()[name]
    b = bsidgen.make_batch(cfg, 0, F)
    d = Decoder.from_config(cfg, b.C, device=0)
    dev = torch.device("cuda", 0)
    rx = torch.from_numpy(b.rx.ravel().copy()).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    rho = torch.from_numpy(b.rho).to(dev)
    L = torch.empty((F, cfg.N, cfg.q), dtype=torch.float32, device=dev)
    st = torch.empty((F,), dtype=torch.int32, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(10):
            d.decode_batch(rx, off, rho, None, L, st, s)
    torch.cuda.synchronize()
    R = 1000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(R):
            d.decode_batch(rx, off, rho, None, L, st, s)
        e1.record(s)
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / R * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        d.decode_batch(rx, off, rho, None, L, st, s)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(R):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / R * 1e3
    res[f"{name}x{F}"] = {"eager_us": eager, "graph_us": graph, "launches": d.last_launch_count()}
    print(f"{name} x {F}: eager {eager:.1f} us/decode, CUDA graph {graph:.1f} us/decode", flush=True)
print(json.dumps(res))
