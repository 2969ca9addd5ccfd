"""One warm-up and one measured launch of the persistent wide sweep kernel at a workload (for ncu:
-k regex:k_sweep_wide -s 1 -c 1)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
nsw = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = synth.CONFIGS[name]
dev = torch.device("cuda:0")
if cfg.numel > 2e8:
    Xd, _, xn = synth.tensor_torch(cfg, device=dev)
    Ad = synth.init_factors_torch(cfg, xn, device=dev)
else:
    X = synth.tensor(cfg)
    Xd = torch.from_numpy(X).to(dev)
    Ad = [torch.from_numpy(a).to(dev) for a in synth.init_factors(cfg, X)]
h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler="leverage", rule=cfg.rule, eta=cfg.eta, seed=1, fused=False)
print("path", h.path)
h.sweep(1)
h.sync()
h.sweep(nsw)
h.sync()
print("ok")
