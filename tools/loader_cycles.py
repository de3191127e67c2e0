"""Variant-build probe: prints skipped_target_slots of one config-2 run (with
SKS_EXP_LOADCLK the loader's clock64 cycles are added << 20)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2003_02200_b200 as sk
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
dem = sk.make_synthetic(sk.SyntheticKind.Fractal, n, n, 10.0, 7)
cfg = sk.RunConfig(ns=180, h0=1.5)
st = sk.EngineStats()
sk.total_viewshed(dem, cfg, st)
st = sk.EngineStats()
sk.total_viewshed(dem, cfg, st)
print(os.environ.get("SKS_LIB", "default"), os.environ.get("SKS_FUSED", "1"), "skipped", st.skipped_target_slots,
      "scan_s", st.scan_seconds)
