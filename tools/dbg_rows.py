"""Row-block runs (run_rows) on a small DEM: parts summed vs the whole map."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_02200_b200 as sk
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dem = sk.make_synthetic(sk.SyntheticKind.Fractal, n, n, 10.0, 7)
cfg = sk.RunConfig(ns=36, h0=1.5)
ctx = sk.Context(0)
whole = ctx.total_viewshed(dem.values, 10.0, cfg, raw=True)
d_dem = torch.from_numpy(dem.values).cuda()
for world in (2, 3, 8):
    tot = np.zeros((n, n))
    for r in range(world):
        d_map = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        ctx.run_rows(d_dem.data_ptr(), n, n, 10.0, cfg, r, world, d_map.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        tot += d_map.cpu().numpy()
    print(world, np.max(np.abs(tot - whole) / np.maximum(np.abs(whole), 1e-30)), flush=True)
