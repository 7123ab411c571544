"""Probe: does running the cfg-2 batch as G concurrent pair groups (one stream
each, one CUDA graph) beat one stream?  Prints ms per grad for G = 1, 2, 4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2106_08817_b200 import engine  # noqa: E402
from paper_2106_08817_b200.synthetic import make_config  # noqa: E402

c = make_config(2)
dt = torch.float32
w = c.weights()
src, tgt, z0 = (torch.as_tensor(a, dtype=dt) for a in (c.source, c.target, c.z0))
B = c.batch
for G in (1, 2, 4):
    per = B // G
    bgs = []
    for g in range(G):
        bg = engine.BatchGrad(per, c.shape, c.n_steps, c.mu, w, c.lam, c.rho, dt)
        bg.load(src[g * per:(g + 1) * per], tgt[g * per:(g + 1) * per], z0[g * per:(g + 1) * per])
        bgs.append(bg)
    streams = [torch.cuda.Stream() for _ in range(G)]

    def run():
        main = torch.cuda.current_stream()
        for s, bg in zip(streams, bgs):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                bg.run(stream=s)
        for s in streams:
            main.wait_stream(s)

    run()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"G={G}: {e0.elapsed_time(e1) / 10:.3f} ms per grad of {B} pairs", flush=True)
    del bgs, graph
    torch.cuda.empty_cache()
