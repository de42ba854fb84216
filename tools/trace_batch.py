"""Phase anatomy of the batched tcgen05 kernel from its %globaltimer trace (CTAs 0..15 =
the first stream block's cluster).  python tools/trace_batch.py [--cfg C4] [--streams 256]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C4")
ap.add_argument("--streams", type=int, default=256)
ap.add_argument("--n", type=int, default=200)
args = ap.parse_args()
cfg = getattr(synth, args.cfg)
hop = 64
g = torch.Generator(device="cuda").manual_seed(1)
cond = torch.rand((args.streams, synth.n_frames_for(args.n, hop), cfg.n_layers, 2 * cfg.residual),
                  generator=g, device="cuda") - 0.5
u = torch.rand((args.streams, args.n), generator=g, device="cuda")
m = Model.from_config(cfg).load(synth.make_weights(cfg, 0)).set_kernel("tc")
m.generate(cond, u, hop)
buf = torch.zeros((32, 16, 32), dtype=torch.int64, device="cuda")
m.set_trace(buf, 100)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
m.generate(cond, u, hop)
e.record()
torch.cuda.synchronize()
print(f"{args.cfg} {args.streams} streams: {s.elapsed_time(e) / args.n * 1e3:.1f} us per step (trace build), "
      f"{cfg.n_layers + 4} phases")
t = buf.cpu().numpy().astype(np.int64)
names = {0: "ph3 start", 12: "prod issued all", 13: "mma 1st chunk in", 14: "mma all issued", 1: "mma done",
         19: "epi start", 16: "epi tmem ld", 17: "epi h stored", 2: "epi end", 3: "after sync",
         8: "ph l+2 start", 9: "l+2 mma done", 10: "l+2 epi end", 11: "l+2 synced", 4: "sampler start", 5: "sampler end",
         6: "sampler synced"}
for c in range(16):
    base = t[:, c, 0]
    if np.all(base == 0):
        continue
    row = []
    for ev in (13, 12, 14, 1, 16, 17, 2, 3):
        v = t[:, c, ev]
        if np.all(v == 0):
            continue
        row.append(f"{names[ev]}={np.median(v - base):6.0f}")
    print(f"cta {c:2d}: " + " ".join(row))
b0 = t[:, 0, 0]
print("sample period (ph3 start to next):", np.median(np.diff(b0)), "ns")
