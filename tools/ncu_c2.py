"""One short C2 generation for profiling (ncu): python tools/ncu_c2.py [--n 3000] [--layers 20]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=3000)
ap.add_argument("--layers", type=int, default=20)
ap.add_argument("--skip", type=int, default=256)
args = ap.parse_args()
cfg = synth.Config(args.layers, 64, args.skip)
m = Model.from_config(cfg).load(synth.make_weights(cfg, 0)).set_kernel("cluster")
cond = torch.from_numpy(synth.make_cond(cfg, synth.n_frames_for(args.n, 64), 0))[None].cuda()
u = torch.from_numpy(synth.make_uniforms(args.n, 0))[None].cuda()
m.generate(cond, u, 64)
torch.cuda.synchronize()
print("done", m.info())
