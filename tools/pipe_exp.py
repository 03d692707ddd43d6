"""Experiment: C4 step as k sub-batches pipelined on two CUDA streams (K6 of one overlapping K4 of the
next) vs the single-batch step.  usage: python tools/pipe_exp.py [C4] [k...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes
from paper_2602_07860_b200 import BlurRenderer
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
ks = [int(x) for x in sys.argv[2:]] or [1, 2, 4]
sc = scenes.make(cfg)
dev = torch.device("cuda:0")
v, c = torch.tensor(sc.verts, device=dev), torch.tensor(sc.colors, device=dev)
tgt = torch.tensor(sc.target, device=dev)
n_norm = int(tgt.numel())
flush = torch.empty(64 * 1024 * 1024, device=dev)
for k in ks:
    parts = np.array_split(np.arange(sc.B), k)
    rs = []
    for p in parts:
        s = sc.subset(list(p))
        rs.append(BlurRenderer(s.faces, s.motion, s.cams, s.H, s.W, s.V, device=dev))
    tg = [tgt[list(p)].contiguous() for p in parts]
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    main = torch.cuda.current_stream()

    def step():
        ev0 = torch.cuda.Event(); ev0.record(main)
        prev = None
        dones, res = [], []
        for i, r in enumerate(rs):
            s = streams[i % 2]
            s.wait_event(ev0)
            if prev is not None:
                s.wait_event(prev)
            with torch.cuda.stream(s):
                out = r.forward(v, c)
                fe = torch.cuda.Event(); fe.record(s)
                loss, g = r.l2_loss_grad(out, tg[i], n_norm=n_norm)
                dv, dc = r.backward(v, c, g, reuse_setup=True)
                de = torch.cuda.Event(); de.record(s)
            prev = fe
            dones.append(de)
            res.append((loss, dv, dc))
        for de in dones:
            main.wait_event(de)
        loss = sum(x[0] for x in res); dv = sum(x[1] for x in res); dc = sum(x[2] for x in res)
        return loss, dv, dc

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main); step(); b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    loss, dv, dc = step()
    print("%s k=%d step %.3f ms (%.1f images/s) loss %.6f |dv| %.6e" % (cfg, k, np.median(ts), sc.B / np.median(ts) * 1e3,
          float(loss), float(dv.norm())), flush=True)
