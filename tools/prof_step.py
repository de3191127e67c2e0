"""Runs the device-resident total viewshed a few times (for ncu / nsight).

  python tools/prof_step.py [--config 2] [--steps 1] [--terrain fractal]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_02200_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--terrain", default="fractal")
a = ap.parse_args()
c = bench.CONFIGS[a.config]
n, ns = c["n"], c["ns"]
cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=c["max_distance"])
dem = bench.make_dem(a.config, a.terrain)
ctx = sk.Context(0)
d_dem = torch.from_numpy(dem).cuda()
d_map = torch.zeros((n, n), dtype=torch.float64, device="cuda")
for i in range(a.steps):
    d_map.zero_()
    st = ctx.run_sectors(d_dem.data_ptr(), n, n, 10.0, cfg, list(range(ns // 2)), d_map.data_ptr(),
                         stream=torch.cuda.current_stream().cuda_stream, want_stats=True)
    print(st)
torch.cuda.synchronize()
