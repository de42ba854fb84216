"""Multi-stream cluster kernel timing: run from a -DDVW_PTRACE=1 build
(tools/ab_build.sh "DVW_PTRACE=1"), C2 with 56 streams; prints, per cluster rank and event, the
median time since CTA 0 drew the item's code and the median interval between consecutive items."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200 import _lib as L  # noqa: E402

S = int(os.environ.get("PT_STREAMS", "56"))
cfg = getattr(synth, os.environ.get("PT_CFG", "C2"))
N, hop = 400, 64
w = synth.make_weights(cfg, 0)
cond, u = synth.make_batch(cfg, N, list(range(S)), hop)
m = L.Model.from_config(cfg).load(w).set_kernel("cluster")
m.generate(torch.from_numpy(cond).cuda(), torch.from_numpy(u).cuda(), hop)
m.sync()
info = m.info()
buf = np.zeros((16, 64, 16), dtype=np.uint64)
rc = L._lib.dvw_diag_ptrace(buf.ctypes.data_as(ctypes.c_void_p))
assert rc == 0, rc
nc = info["chain_ctas"]
print("streams", S, "per cluster", info["streams_per_cluster"], "grid", info["last_grid"], "chain", nc)
t = buf.astype(np.float64)
ref = t[0, :, 7]  # CTA 0 drew the item's code (item = sample n of stream s: its code n-1)
names_chain = {0: "A pre ok", 1: "A hin/draw ok", 2: "A L0 gate", 3: "A L1 gate", 4: "A L2 gate", 5: "A L3 gate",
               6: "A0 logits in", 7: "A0 drawn", 8: "X retire", 9: "X last h", 10: "X bar_done", 11: "X release",
               12: "X make_pre end", 13: "B item end", 14: "C xin ok"}
names_head = {0: "h(l-1) in", 1: "h(l) in", 2: "partials in", 4: "z_a in", 5: "logits sent"}
names_skip = {0: "first h in", 1: "last h in", 2: "partial sent"}
size = info["last_cluster"]
for r in range(size):
    role = "chain" if r < nc else ("head" if r < nc + 4 else "skip")
    names = names_chain if role == "chain" else (names_head if role == "head" else names_skip)
    out = []
    for ev, nm in names.items():
        col = t[r, :, ev]
        ok = (col > 0) & (ref > 0)
        if ok.sum() < 8:
            continue
        rel = np.median((col - ref)[ok]) / 1e3
        d = np.diff(col[col > 0])
        per = np.median(d) / 1e3 if d.size else float("nan")
        out.append(f"{nm} {rel:+.2f}/{per:.2f}")
    print(f"rank {r:2d} {role:5s} | " + " | ".join(out))
print("(us: median since CTA 0 drew the item / median interval between consecutive items)")
