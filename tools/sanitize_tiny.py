"""Tiny invocations of every kernel family for compute-sanitizer (SURVEY.md §5 race detection).

    compute-sanitizer --tool racecheck python tools/sanitize_tiny.py --kernel cluster

Each run checks its codes against the CPU oracle too (a race that changes results fails here
even if the tool misses it)."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: the check only)
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Conditioner, Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kernel", default="cluster",
                choices=["cluster", "cluster_pipe", "cluster_pipe40", "stream", "tc", "parallel", "conditioner"])
args = ap.parse_args()

hop = 8
if args.kernel == "conditioner":
    cw = synth.make_conditioner_weights(32, 16, 4, 64, 0)
    c = Conditioner(32, 16, 4, 64).load(cw)
    f = torch.from_numpy(synth.make_features(24, 32, 0))[None].cuda()
    out = c.run(f)
    torch.cuda.synchronize()
    print("conditioner ok", tuple(out.shape), float(out.abs().max()))
    sys.exit(0)

cfg = synth.Config(4, 64, 128) if args.kernel != "tc" else synth.Config(2, 64, 128)
N = 48 if args.kernel != "tc" else 12
S = 2 if args.kernel in ("tc", "cluster") else 1
kern = args.kernel
if args.kernel == "cluster_pipe":  # multi-stream variant, LP = 3: 5 streams, 4 per cluster (ragged)
    S, kern = 5, "cluster"
    os.environ["DVW_CLUSTER_W"] = "4"
elif args.kernel == "cluster_pipe40":  # multi-stream variant, LP = 4 with chain-skip batches (l = 40)
    cfg, N, S, kern = synth.C3, 12, 3, "cluster"
    os.environ["DVW_CLUSTER_W"] = "3"
w = synth.make_weights(cfg, 0)
cond, u = synth.make_batch(cfg, N, list(range(S)), hop)
m = Model.from_config(cfg).load(w).set_kernel(kern)
dc, du = torch.from_numpy(cond).cuda(), torch.from_numpy(u).cuda()
if args.kernel == "parallel":
    codes = np.stack([synth.make_codes(N, s) for s in range(S)])
    lg = m.logits(dc, torch.from_numpy(codes).cuda(), hop).cpu().numpy()
    _, ref, _ = oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond[0], hop, N, forced=codes[0])
    err = float(np.max(np.abs(lg[0] - ref)))
    assert err < 2e-5, err
    print("parallel ok", err)
else:
    codes = m.generate(dc, du, hop).cpu().numpy()
    m.sync()
    for s in range(S):
        ref, _, _ = oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond[s], hop, N, uniforms=u[s],
                               dilations=cfg.dilation_list())
        assert np.array_equal(codes[s], ref), s
    print(args.kernel, "ok", m.info())
