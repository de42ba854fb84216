"""Teacher-forced logits (dvw_logits) for one utterance: the parallel-over-time kernel vs the
autoregressive cluster kernel in teacher-forced mode.  python tools/bench_logits.py [--cfg C2]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.environ.get("DVW_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C2")
ap.add_argument("--n", type=int, default=16000)
ap.add_argument("--streams", type=int, default=1)
args = ap.parse_args()
cfg = getattr(synth, args.cfg)
hop = 64
cond, _ = synth.make_batch(cfg, args.n, list(range(args.streams)), hop)
codes = torch.stack([torch.from_numpy(synth.make_codes(args.n, u)) for u in range(args.streams)]).cuda()
cond = torch.from_numpy(cond).cuda()
m = Model.from_config(cfg).load(synth.make_weights(cfg, 0))


def timeit(kernel, reps=5):
    m.set_kernel(kernel)
    m.logits(cond, codes, hop)
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        m.logits(cond, codes, hop)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best, m.info()


macs = cfg.n_layers * (5 * cfg.residual ** 2 + cfg.residual * cfg.skip) + 256 * cfg.skip + 256 * 256
out = {"cfg": args.cfg, "samples": args.n, "streams": args.streams}
for k in ("parallel", "cluster" if args.streams == 1 and cfg.residual == 64 else "tc"):
    ms, info = timeit(k)
    tflops = 2.0 * macs * args.n * args.streams / (ms * 1e-3) / 1e12
    out[k] = {"ms": ms, "samples_per_s": args.n * args.streams / (ms * 1e-3), "tflops": tflops,
              "launches": info["last_launches"]}
print(json.dumps(out))
