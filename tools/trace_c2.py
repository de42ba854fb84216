"""Per-sample timeline of the batch-1 cluster kernel from its %globaltimer trace.

    python tools/trace_c2.py [--layers 20] [--skip 256] [--n 4000] [--first 3000] [--count 64]

Prints, averaged over the traced samples, each CTA's event times relative to the
start of the sample on chain CTA 0 (ns), and the per-layer clock64 spans of every
chain CTA (cycles).  Event ids: see kernel_cluster.cu (trace / trace_clk calls).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("DVW_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=20)
ap.add_argument("--skip", type=int, default=256)
ap.add_argument("--n", type=int, default=4000)
ap.add_argument("--first", type=int, default=3000)
ap.add_argument("--count", type=int, default=64)
args = ap.parse_args()

cfg = synth.Config(args.layers, 64, args.skip)
w = synth.make_weights(cfg, 0)
hop = 64
cond = torch.from_numpy(synth.make_cond(cfg, synth.n_frames_for(args.n, hop), 0))[None].cuda()
u = torch.from_numpy(synth.make_uniforms(args.n, 0))[None].cuda()
m = Model.from_config(cfg).load(w)
m.generate(cond, u, hop)
torch.cuda.synchronize()
buf = torch.zeros((args.count, 16, 32), dtype=torch.int64, device="cuda")
m.set_trace(buf, args.first)
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
m.generate(cond, u, hop)
en.record()
torch.cuda.synchronize()
print(f"traced run: {st.elapsed_time(en) / args.n * 1e3:.3f} us/sample (trace build)")
m.set_trace(None)
t = buf.cpu().numpy().astype(np.int64)
info = m.info()
ncta = info["last_cluster"]
base = t[:, 0, 0].copy()  # chain CTA 0, event 0: start of the sample's first layer
period = np.diff(base)
print(f"sample period {np.median(period):.0f} ns (median), min {period.min()} max {period.max()}")
c0 = t[:, 0, :]
if not np.all(c0[:, 1] == 0):
    d = lambda a, b: np.median(c0[:, b] - c0[:, a])  # noqa: E731
    print(f"CTA 0 sampler (cycles): logits-in -> call {d(1, 4):.0f}, sample_warp {d(4, 6):.0f}, "
          f"-> embed stored {d(6, 7):.0f}, -> barrier passed {d(7, 30):.0f}, -> layer 0 start {d(30, 8):.0f}")
names = {0: "start/recv", 1: "q/partial", 2: "za/done", 3: "logits", 4: "h[l-1] in", 5: "pre ready", 6: "d2 done", 7: "zs sync", 9: "za sent", 20: "sampled"}
for c in range(ncta):
    row = []
    for ev in (4, 6, 0, 1, 7, 9, 2, 3, 5, 20):
        v = t[:, c, ev]
        if np.all(v == 0):
            continue
        d = v - base
        row.append(f"{names[ev]}={np.median(d):7.0f}")
    cyc = []
    for jl in range(3):
        a, b = t[:, c, 8 + 2 * jl], t[:, c, 9 + 2 * jl]
        if np.all(a == 0):
            continue
        cyc.append(f"L{jl}:{np.median(b - a):.0f}")
    if c < 7:
        for jl in range(3):
            st, bra, ara, gate, cra, bh = (t[:, c, e] for e in (8 + 2 * jl, 14 + jl, 17 + jl, 27 + jl, 21 + jl, 24 + jl))
            if np.all(st == 0):
                continue
            parts = [f"L{jl}:"]
            if not np.all(bra == 0):
                parts.append(f"toRA={np.median(bra - st):.0f} waitRA={np.median(ara - bra):.0f} Carr={np.median(cra - st):.0f}")
            parts.append(f"gate@{np.median(gate - st):.0f}")
            if not np.all(bh == 0):
                parts.append(f"Barr(prev h)={np.median(bh - st):.0f}")
            cyc.append(" ".join(parts))
    gaps = []
    for jl in range(2):
        a, b = t[:, c, 9 + 2 * jl], t[:, c, 8 + 2 * (jl + 1)]
        if np.all(b == 0):
            continue
        gaps.append(f"g{jl}:{np.median(b - a):.0f}")
    print(f"cta {c:2d}: " + " ".join(row) + ("  cyc " + " ".join(cyc + gaps) if cyc else ""))
