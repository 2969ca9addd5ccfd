"""Phase timeline of the persistent wide sweep kernel (k_sweep_wide) at a workload: globaltimer marks
of CTA 0 (CPSGD_DEBUG_TIMERS), per iteration: S(ample) | bar | G(ather) | bar | U(pdate) | bar |
P(airs) | I(nverse) | Q (scores/scan) | bar.  Also us/sweep of the persistent kernel and the chain."""
import os
import sys

os.environ["CPSGD_DEBUG_TIMERS"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04081_b200 import CPSGD  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    sampler = sys.argv[2] if len(sys.argv) > 2 else "leverage"
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda:0")
    if cfg.numel > 2e8:
        Xd, _, xn = synth.tensor_torch(cfg, device=dev)
        Ad0 = synth.init_factors_torch(cfg, xn, device=dev)
    else:
        X = synth.tensor(cfg)
        A0 = synth.init_factors(cfg, X)
        Xd = torch.from_numpy(X).to(dev)
        Ad0 = [torch.from_numpy(a).to(dev) for a in A0]
    for persist in ((True,) if os.environ.get("CPSGD_PW_ABLATE") else (True, False)):
        Ad = [a.clone() for a in Ad0]
        h = CPSGD(Xd, cfg.dims, Ad, cfg.batch, sampler=sampler, rule=cfg.rule, eta=cfg.eta, seed=1, fused=False,
                  persist=persist)
        h.sweep(3)
        h.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        h.sweep(20)
        e1.record(h.stream)
        h.sync()
        print(h.path, "us/sweep", round(e0.elapsed_time(e1) * 1e3 / 20, 2), flush=True)
        if persist:
            h.sweep(3)
            h.sync()
            dt = h.debug_timers()
            d = np.concatenate([np.array(dt[512:512 + 256], dtype=np.int64).reshape(8, 32),
                                np.array(dt[3072:3072 + 256], dtype=np.int64).reshape(8, 32)], axis=1)  # 32+: PW_MK2
            # marks: 0 start, 11 cdf staged, 12 draws, 13 skr, 14 gamma, 1 S end, 2 bar, 3 G end, 4 bar,
            # 15 U loads, 16 U update, 5 U end, 6 bar, 7 P end, 18 pair wait, 19 gram load, 20 inverse,
            # 21 scores, 22 lookback, 8 I+Q end, 9, 10 bar
            seq = [("S:wait", 0, 38), ("S:stage", 38, 11), ("S:d-entry", 11, 32), ("S:d-philox", 32, 33), ("S:d-search", 33, 34), ("S:d-div", 34, 35), ("S:d-sync", 35, 36), ("S:weights", 36, 12), ("S:skr", 12, 13), ("S:img", 13, 23), ("S:gblk", 23, 24), ("S:gred", 24, 14), ("S:tail", 14, 1),
                   ("barS", 1, 2), ("G:sfb", 2, 25), ("G:first", 25, 26), ("G:stream", 26, 27), ("G:mma", 27, 28),
                   ("G:epi", 28, 29), ("G:tail", 29, 3), ("barG", 3, 4), ("U:issue+M", 4, 39), ("U:cpwait", 39, 40), ("U:gamwait", 40, 41), ("U:sync", 41, 15), ("U:upd", 15, 16),
                   ("U:gram", 16, 5), ("barU", 5, 6), ("P", 6, 7), ("I:wait", 7, 18), ("I:load", 18, 19),
                   ("I:inv", 19, 20), ("Q:score", 20, 21), ("Q:tail", 21, 9),
                   ("barQ", 9, 10)]
            rows = []
            for s in range(1, 8):
                t = d[s]
                if t[0] == 0 or t[10] == 0:
                    continue
                rows.append([t[b] - t[a] if t[a] and t[b] else 0 for _, a, b in seq])
            # marks are clock64 cycles (slots 30/31: globaltimer ns at marks 0/10): cycles -> us
            ghz = float(np.mean([(d[s, 10] - d[s, 0]) / (d[s, 31] - d[s, 30]) for s in range(1, 8)]))
            rows = np.array(rows) / ghz / 1e3
            print("phase us (CTA 0, mean over iterations 1..7):")
            for (nm, _, _), v in zip(seq, rows.mean(0)):
                print(f"  {nm:8s} {v:8.2f}")

            print("  total", round(float((d[1:8, 31] - d[1:8, 30]).mean()) / 1e3, 2), "us; SM clock", round(ghz * 1e3), "MHz")
        h.close()
        del Ad
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
