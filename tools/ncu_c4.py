"""One short C4 (256 streams, batched tcgen05 kernel) generation for ncu: python tools/ncu_c4.py [--n 200]"""
import argparse
import os
import sys

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
cond, u = synth.make_batch_hashed_torch(cfg, args.n, list(range(args.streams)), 64, torch.device("cuda"))
m = Model.from_config(cfg).load(synth.make_weights(cfg, 0)).set_kernel("tc")
m.generate(cond, u, 64)
torch.cuda.synchronize()
print("done", m.info())
