"""Independent chains side by side on one GPU (SURVEY 8(f).2 on the persistent path): K handles on the same
resident tensor, each planned for 148 / K SMs (CPSGD_SMS), their cooperative sweep launches on K streams.
Prints us/sweep of one chain at 148 and at 148 / K SMs, and the aggregate fibers/s of K concurrent chains.
python tools/pw_multi.py [C4] [K] [sweeps]"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
S = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cfg = synth.CONFIGS[name]
dev = torch.device("cuda:0")
Xd, _, xn = synth.tensor_torch(cfg, device=dev)
A0 = synth.init_factors_torch(cfg, xn, device=dev)
fps = cfg.order * cfg.batch


def timed(hs, streams, sweeps):
    for h in hs:
        h.sweep(3)
    for h in hs:
        h.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    ev = []
    for st in streams:  # every chain starts after e0
        st.wait_event(e0)
    for h in hs:
        h.sweep(sweeps)
    for st in streams:
        x = torch.cuda.Event()
        x.record(st)
        ev.append(x)
    for x in ev:
        torch.cuda.current_stream().wait_event(x)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    for h in hs:
        h.sync()
    return e0.elapsed_time(e1) * 1e3  # us


for sms in (148, 148 // K):
    os.environ["CPSGD_SMS"] = str(sms)
    st = torch.cuda.Stream()
    Ad = [a.clone() for a in A0]
    with torch.cuda.stream(st):
        h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler="leverage", rule=cfg.rule, eta=cfg.eta, seed=1, fused=False,
                  stream=st)
    t = timed([h], [st], S)
    print(f"one chain, {sms} SMs: path {h.path}, {t / S:.2f} us/sweep, {fps * S / (t * 1e-6) / 1e6:.2f} M fibers/s",
          flush=True)
    h.close()
    del Ad
    torch.cuda.empty_cache()

os.environ["CPSGD_SMS"] = str(148 // K)
hs, sts, Ads = [], [], []
for c in range(K):
    st = torch.cuda.Stream()
    Ad = [a.clone() for a in A0]
    with torch.cuda.stream(st):
        hs.append(CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler="leverage", rule=cfg.rule, eta=cfg.eta, seed=1 + c,
                        fused=False, stream=st))
    sts.append(st)
    Ads.append(Ad)
t = timed(hs, sts, S)
print(f"{K} chains x {148 // K} SMs concurrently: paths {[h.path for h in hs]}, {t / S:.2f} us per sweep of all, "
      f"{K * fps * S / (t * 1e-6) / 1e6:.2f} M fibers/s aggregate", flush=True)
