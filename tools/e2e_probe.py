import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, synth
from paper_2103_04081_b200 import CPSGD
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
dev = torch.device("cuda:0")
Xd, _, xn = synth.tensor_torch(cfg, device=dev)
Ad = synth.init_factors_torch(cfg, xn, device=dev)
h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler="leverage", rule=cfg.rule, alpha=cfg.alpha, eta=cfg.eta, seed=0)
h.sweep(5); h.sync()
host = [a.detach().cpu().pin_memory() for a in Ad]
for it in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.steps_host(0, len(cfg.dims), host)
    t1 = time.perf_counter()
    print(f"call {it}: {(t1 - t0) * 1e3:.3f} ms")
h.profile(True)
h.steps_host(0, len(cfg.dims), host)
print(h.profile_read())
h.profile(False)
# the pieces on the device clock: pinned copies in / out, one sweep
st = h.stream
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for _ in range(3):
    e[0].record(st)
    with torch.cuda.stream(st):
        for a, b in zip(Ad, host):
            a.copy_(b, non_blocking=True)
    e[1].record(st)
    h.sweep(1)
    e[2].record(st)
    with torch.cuda.stream(st):
        for a, b in zip(Ad, host):
            b.copy_(a, non_blocking=True)
    e[3].record(st)
    torch.cuda.synchronize()
    print(f"H2D {e[0].elapsed_time(e[1]) * 1e3:.1f} us, sweep {e[1].elapsed_time(e[2]) * 1e3:.1f} us, "
          f"D2H {e[2].elapsed_time(e[3]) * 1e3:.1f} us")
