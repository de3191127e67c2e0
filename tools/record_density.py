"""Offline model: in the target-lockstep scan (64-POV tasks, 16-target windows
after the exact-bound skip), how often does a 4-target group contain a
near-hit/record for ANY of the task's 64 POVs? (Decides whether a
branch-on-any-candidate inner loop pays.) FP64 emulation, band ignored."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2003_02200_b200 as sk
from _oracle import Orc

orc = Orc()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
dem = sk.make_synthetic(sk.SyntheticKind.Fractal, n, n, 10.0, 7).values
rng = np.random.default_rng(1)
tot = dict(groups=0, any_group=0, win=0, win_eval=0, pairs=0, rec=0, any8=0, groups8=0)
for ksec in (3, 20, 41, 66):
    p = orc.plan_sector(ksec, 180, n, n)
    g = orc.apply_pre_ops(dem, ksec, 180)
    vals, w, rr, base = orc.build_skw(g, p.shear_tan)
    rows = [q for q in range(len(rr)) if rr[q][1] - rr[q][0] > 200]
    for q in rng.choice(rows, 4, replace=False):
        a, b = rr[q]
        row = vals[q, a:b].astype(np.float64)
        L = len(row)
        for d in (0, 1):
            r = row if d == 0 else row[::-1]
            for c in range(0, L, 64):
                ys = np.arange(c, min(c + 64, L))
                h = r[ys] + 1.5
                mx = np.full(len(ys), -np.inf)
                # windows of 16 from c
                for k0 in range(c, L, 16):
                    ks = np.arange(k0, min(k0 + 16, L))
                    dd = ks[None, :] - ys[:, None]
                    valid = dd >= 1
                    th = np.where(valid, (r[ks][None, :] - h[:, None]) / np.where(valid, dd, 1), -np.inf)
                    tot["win"] += 1
                    # skip test (exact bound of the window): max over window < running max for all POVs
                    ub = th.max(axis=1)
                    if k0 >= c + 64 and np.all(ub < mx):
                        continue
                    tot["win_eval"] += 1
                    for gi in range(0, len(ks), 4):
                        sub = th[:, gi:gi + 4]
                        recs = np.zeros_like(sub, dtype=bool)
                        for t in range(sub.shape[1]):
                            rec = sub[:, t] > mx
                            recs[:, t] = rec
                            mx = np.where(rec, sub[:, t], mx)
                        tot["groups"] += 1
                        tot["pairs"] += int(valid[:, gi:gi + 4].sum())
                        tot["rec"] += int(recs.sum())
                        tot["any_group"] += int(recs.any())
                        # a finer unit: 8 POVs (4 lanes) x 4 targets
                        for l8 in range(0, recs.shape[0], 8):
                            tot["groups8"] += 1
                            tot["any8"] += int(recs[l8:l8 + 8].any())
print(tot)
print("evaluated windows %.3f, record density %.4f, groups with any record (64 POVs) %.3f, per 8 POVs %.3f" % (
    tot["win_eval"] / tot["win"], tot["rec"] / max(tot["pairs"], 1), tot["any_group"] / tot["groups"],
    tot["any8"] / tot["groups8"]))
