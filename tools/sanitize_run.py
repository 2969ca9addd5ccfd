"""A small run of one execution path, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
python tools/sanitize_run.py fused|chain|persistent|sharded|replica [f32|f64]
Each path: init (tables), two cyclic sweeps + one step, fit, all through the C ABI; exits 0 when the
library reports no error.  Shapes are ragged (partial tiles / units / chunks)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402
from paper_2103_04081_b200.cpsgd import nccl_unique_id  # noqa: E402

path = sys.argv[1]
dt = sys.argv[2] if len(sys.argv) > 2 else "f32"
dev = torch.device("cuda:0")
if path == "fused":
    cfg = synth.small((60, 44, 37), 8, dtype=dt, batch=200, rule="adaptive", eta=0.05, seed=1)
else:
    cfg = synth.small((300, 130, 70), 20, dtype=dt, batch=1000, rule="adaptive", eta=0.03, seed=1)
X = synth.tensor(cfg)
A0 = synth.init_factors(cfg, X)
Xd = torch.from_numpy(X).to(dev)
Ad = [torch.from_numpy(a.copy()).to(dev) for a in A0]
kw = dict(sampler="leverage", rule=cfg.rule, eta=cfg.eta, seed=3)
if path == "fused":
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, **kw)
elif path == "chain":
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, fused=False, persist=False, **kw)
elif path == "persistent":
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, fused=False, **kw)
elif path == "sharded":
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, fused=False, force_comm=True, nccl_id=nccl_unique_id(), **kw)
elif path == "replica":
    h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, fused=False, replica=True, force_comm=True, nccl_id=nccl_unique_id(), **kw)
else:
    raise SystemExit("unknown path " + path)
print("path", h.path, flush=True)
h.sweep(2)
h.step(0)
h.sync()
f = h.fit()
assert np.isfinite(f), f
assert all(torch.isfinite(a).all() for a in Ad)
h.close()
print("ok", path, dt, "fit", f)
