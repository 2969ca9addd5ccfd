"""Gather-kernel HBM efficiency vs batch size on the C4 tensor (2000^3 fp32, R = 50).

The tcgen05 gather kernel moves B x I_n x 4 bytes per launch (32.8 MB at C4's B = 4096): launch,
prologue, epilogue and tail are a fixed cost, so its fraction of the HBM roofline grows with the
batch.  Prints one line per batch: CUDA-event duration of k_gather_update_tc (direct launches),
algorithmic GB/s and the fraction of MEASURED_PEAKS.json's copy bandwidth.  (A measurement of the
kernel, not a bench line: the bench's C4 uses BASELINE's B = 4096.)
"""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
base = synth.CONFIGS["C4"]
dev = torch.device("cuda:0")
Xd, _, xn = synth.tensor_torch(base, device=dev)
A0 = synth.init_factors_torch(base, xn, device=dev)
for B in [int(a) for a in (sys.argv[1:] or ["4096", "16384", "65536"])]:
    cfg = dataclasses.replace(base, batch=B)
    Ad = [a.clone() for a in A0]
    h = CPSGD(Xd, cfg.dims, Ad, B, sampler="leverage", rule=cfg.rule, eta=cfg.eta, seed=0)
    h.sweep(1)
    h.sync()
    h.profile(True)
    h.sweep(3)
    prof = h.profile_read()
    h.profile(False)
    if "k_gather_update_tc" not in prof:
        print(f"B={B:6d}: not on the tcgen05 wide path ({sorted(prof)})")
        h.close()
        continue
    t, c = prof["k_gather_update_tc"]
    us = 1e3 * t / c
    gbs = B * cfg.dims[0] * 4 / (us * 1e-6) / 1e9
    print(f"B={B:6d}: k_gather_update_tc {us:7.1f} us, {gbs:7.1f} GB/s algorithmic = {100 * gbs / peak:5.1f} % of "
          f"{peak:.0f} GB/s; kernels: " + ", ".join(f"{k} {1e3 * v[0] / v[1]:.1f}" for k, v in prof.items()))
    h.close()
    del Ad
    torch.cuda.empty_cache()
