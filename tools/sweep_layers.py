"""Untraced per-sample time of the batch-1 cluster kernel vs layer count (slope = per-layer
cost including the amortised hops).  python tools/sweep_layers.py [--skip 256] [--n 8000]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.environ.get("DVW_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--skip", type=int, default=256)
ap.add_argument("--n", type=int, default=8000)
ap.add_argument("--layers", default="1,2,4,8,12,16,20,24,28,32,36,40")
args = ap.parse_args()
hop = 64
for L in [int(x) for x in args.layers.split(",")]:
    cfg = synth.Config(L, 64, args.skip)
    try:
        m = Model.from_config(cfg).load(synth.make_weights(cfg, 0)).set_kernel("cluster")
    except Exception as e:  # noqa: BLE001
        print(f"L={L:3d}: {e}")
        continue
    cond = torch.from_numpy(synth.make_cond(cfg, synth.n_frames_for(args.n, hop), 0))[None].cuda()
    u = torch.from_numpy(synth.make_uniforms(args.n, 0))[None].cuda()
    m.generate(cond, u, hop)
    best = 1e9
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        m.generate(cond, u, hop)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) * 1e3 / args.n)
    info = m.info()
    print(f"L={L:3d}: {best:7.3f} us/sample  cluster={info['last_cluster']}", flush=True)
