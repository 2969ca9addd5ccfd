"""Marginal cost of each phase of the persistent wide kernel on the critical path: us/sweep with phases
switched off (CPSGD_PW_ABLATE_MASK, results garbage -- timing only).  python tools/pw_ablate.py [C4|C2]"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
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
assert h.path == "persistent"
# sensitivity experiments that keep the data path sane (results stay finite): doubled work, stale images
MASKS = [(0, "full"), (0x120, "MMA twice"), (0x140, "split twice"),
         (0x180, "no A-image copies (stale)"), (0x102, "no fiber loads"), (0, "full again")]
if len(sys.argv) > 2 and sys.argv[2] == "destructive":  # garbage data: indicative only
    MASKS = [(0, "full"), (0x101, "no inverse (W = diag)"), (0x102, "no fiber loads"), (0x104, "no pair sums / Gram load"),
             (0x108, "no update Gram partials"), (0x110, "no scores"), (0x105, "no P + inverse"),
             (0x11f, "all of the above off")]
for mask, what in MASKS:
    os.environ["CPSGD_PW_ABLATE_MASK"] = str(mask)
    h.sweep(3)
    h.sync() if mask == 0 else torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(h.stream)
    h.sweep(20)
    e1.record(h.stream)
    torch.cuda.synchronize()
    print(f"{mask:#06x} {what:28s} {e0.elapsed_time(e1) * 1e3 / 20:8.2f} us/sweep", flush=True)
