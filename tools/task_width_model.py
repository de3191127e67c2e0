"""Offline model: fraction of (POV, target) slots the target-lockstep scan
evaluates (16-target windows, exact-bound skip after the first 64 targets of
a task) for task widths of 64 vs 32 POVs, incl. the dead triangle slots."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2003_02200_b200 as sk
from _oracle import Orc

orc = Orc()
n = 2000
dem = sk.make_synthetic(sk.SyntheticKind.Fractal, n, n, 10.0, 7).values
rng = np.random.default_rng(1)
res = {}
for W, NT in ((64, 64), (32, 64), (32, 32)):
    ev = tot = useful = 0
    for ksec in (3, 20, 41, 66):
        p = orc.plan_sector(ksec, 180, n, n)
        g = orc.apply_pre_ops(dem, ksec, 180)
        vals, w, rr, base = orc.build_skw(g, p.shear_tan)
        rows = [q for q in range(len(rr)) if rr[q][1] - rr[q][0] > 200]
        for q in np.random.default_rng(ksec).choice(rows, 3, replace=False):
            a, b = rr[q]
            row = vals[q, a:b].astype(np.float64)
            L = len(row)
            for d in (0, 1):
                r = row if d == 0 else row[::-1]
                for c in range(0, L, W):
                    ys = np.arange(c, min(c + W, L))
                    h = r[ys] + 1.5
                    mx = np.full(len(ys), -np.inf)
                    for k0 in range(c, L, 16):
                        ks = np.arange(k0, min(k0 + 16, L))
                        dd = ks[None, :] - ys[:, None]
                        valid = dd >= 1
                        th = np.where(valid, (r[ks][None, :] - h[:, None]) / np.where(valid, dd, 1), -np.inf)
                        tot += W * len(ks)
                        useful += int(valid.sum())
                        ub = th.max(axis=1)
                        if k0 >= c + NT and np.all(ub < mx):
                            continue
                        ev += W * len(ks)
                        for t in range(th.shape[1]):
                            rec = th[:, t] > mx
                            mx = np.where(rec, th[:, t], mx)
    res[W] = (ev, tot, useful)
    print(W, NT, "evaluated slots / useful pairs = %.4f" % (ev / useful), "evaluated/all slots %.4f" % (ev / tot))
