"""Print the cluster plan's co-resident cluster counts (dvw_info) for C1/C2/C3 on this GPU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_07825_b200 import synth  # noqa: E402
from paper_1702_07825_b200._lib import Model  # noqa: E402
for name in ("C1", "C2", "C3"):
    cfg = getattr(synth, name)
    m = Model.from_config(cfg).load(synth.make_weights(cfg, 0))
    i = m.info()
    print(name, {k: i[k] for k in ("chain_ctas", "max_clusters", "max_clusters_pipe")}, flush=True)
