"""Multi-stream cluster kernel vs the oracle for a few W / configs; prints the first mismatch."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Model  # noqa: E402

def run(cfg, S, W, N, lp=None):
    if lp: os.environ["DVW_CLUSTER_LP"] = str(lp)
    else: os.environ.pop("DVW_CLUSTER_LP", None)
    hop = 64
    w = synth.make_weights(cfg, 0)
    cond, u = synth.make_batch(cfg, N, list(range(S)), hop)
    m = Model.from_config(cfg).load(w).set_kernel("cluster")
    os.environ["DVW_CLUSTER_W"] = str(W)
    codes = m.generate(torch.from_numpy(cond).cuda(), torch.from_numpy(u).cuda(), hop).cpu().numpy()
    m.sync()
    res = []
    for st in range(S):
        ref, _, _ = oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond[st], hop, N, uniforms=u[st],
                               dilations=cfg.dilation_list(), want_logits=False)
        d = np.nonzero(codes[st] != ref)[0]
        res.append(int(d[0]) if d.size else -1)
    print(f"l={cfg.n_layers} lp={lp} S={S} W={W} N={N}: first mismatch per stream {res}", flush=True)

run(synth.C3, 9, 8, 160)
run(synth.C3, 6, 3, 160)
run(synth.C3, 5, 2, 160)
run(synth.C2, 8, 8, 160, lp=4)
run(synth.C2, 20, 8, 160, lp=3)
