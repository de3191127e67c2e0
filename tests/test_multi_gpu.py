"""Multi-GPU paths: the in-process C ABI (sks_total_viewshed_devices /
RunConfig.n_gpus: one host thread per GPU, one NCCL reduce) and the
one-process-per-GPU torch.distributed path (mode="rows" + RowBalancer),
against the reference.

The pool's boxes have ONE B200, so the sharding is exercised with ranks that
share it: a device list with repeats ([0, 0], [0, 0, 0]) reduces with peer
adds, and NCCL itself runs as a one-rank communicator (SKS_NCCL=1). The
reference's analogue is worker-count determinism (acceptance_main.cpp:255-277,
test_engine.cpp:53-64); across GPUs only the per-cell summation order
differs, so the bar is 1e-12 relative (the reference's is 1e-5), and one
rank is bit-exact.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2003_02200_b200 as sk
from _oracle import Orc, Ref, have_ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def b64(a):
    return np.ascontiguousarray(a).view(np.uint64)


def _ora():
    return Ref() if have_ref() else Orc()


# ---- host logic (CPU) -------------------------------------------------------------

def _cuts_update_restated(cuts, times):
    """Plain restatement of the rebalancing step (time piecewise linear in the
    cost fraction; new cuts at equal shares of the total time)."""
    c = np.asarray(cuts, np.float64)
    t = np.asarray(times, np.float64)
    n = len(t)
    T = np.concatenate([[0.0], np.cumsum(t)])
    if not np.all(np.isfinite(t)) or np.any(t < 0) or T[-1] <= 0:
        return c.copy()
    new = [0.0]
    for b in range(1, n):
        target = b * T[-1] / n
        r = int(np.searchsorted(T, target, side="right") - 1)
        r = min(max(r, 0), n - 1)
        frac = (target - T[r]) / t[r] if t[r] > 0 else 0.0
        new.append(c[r] + min(max(frac, 0.0), 1.0) * (c[r + 1] - c[r]))
    new.append(1.0)
    return np.maximum.accumulate(np.clip(np.asarray(new), 0.0, 1.0))


def test_row_cuts_update_matches_restatement():
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 8):
        cuts = np.linspace(0, 1, n + 1)
        for _ in range(50):
            times = rng.random(n) * 10
            if rng.random() < 0.1:
                times[rng.integers(0, n)] = 0.0
            got = sk.row_cuts_update(cuts, times)
            assert np.array_equal(got, _cuts_update_restated(cuts, times))
            assert got[0] == 0.0 and got[-1] == 1.0 and np.all(np.diff(got) >= 0)
            cuts = got


def test_row_cuts_update_balances_linear_costs():
    """When time really is piecewise linear in the cost fraction (a constant
    density per old block), one step gives every new block the same time."""
    dens = np.array([1.0, 3.0, 2.0, 0.5])
    cuts = np.array([0.0, 0.2, 0.45, 0.8, 1.0])
    times = dens * np.diff(cuts)
    new = sk.row_cuts_update(cuts, times)
    F = lambda x: np.interp(x, cuts, np.concatenate([[0.0], np.cumsum(times)]))  # noqa: E731
    block = np.diff([F(x) for x in new])
    np.testing.assert_allclose(block, times.sum() / 4, rtol=1e-12)


def test_gpu_count_is_validated_like_workers():
    """validate(RunConfig) rejects workers < 1 (dem.cpp:74-78); n_gpus takes
    its place (-1 = every visible GPU)."""
    dem = sk.make_synthetic(sk.SyntheticKind.Flat, 4, 4, 10.0)
    with pytest.raises(ValueError, match="GPU count must be >= 1"):
        sk.validate(dem, sk.RunConfig(n_gpus=0))
    sk.validate(dem, sk.RunConfig(n_gpus=sk.ALL_GPUS))
    sk.validate(dem, sk.RunConfig(n_gpus=8))


def test_config_devices():
    assert sk.config_devices(sk.RunConfig()) == [0]
    assert sk.config_devices(sk.RunConfig(device=2)) == [2]
    assert sk.config_devices(sk.RunConfig(device=1, n_gpus=3)) == [1, 2, 3]
    # every visible device (at least the first one named)
    n = sk.device_count()
    assert sk.config_devices(sk.RunConfig(n_gpus=sk.ALL_GPUS)) == list(range(max(1, n)))


# ---- in-process multi-GPU on the device -----------------------------------------------

@pytest.mark.gpu
def test_devices_one_gpu_bitexact():
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 48, 40, 10.0, 13)
    cfg = sk.RunConfig(ns=36, h0=1.5, units=sk.Units.SquareMeters)
    ref = _ora().total_viewshed(dem.values, 10.0, 36, 1.5, raw=True)
    assert np.array_equal(b64(sk.total_viewshed_devices(dem, cfg, [0], raw=True)), b64(ref))
    # n_gpus = ALL on a one-GPU box is the same single-device run
    cfg_all = sk.RunConfig(ns=36, h0=1.5, units=sk.Units.SquareMeters, n_gpus=sk.ALL_GPUS)
    if sk.device_count() == 1:
        assert np.array_equal(b64(sk.total_viewshed_raw(dem, cfg_all)), b64(ref))


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0, 0, 0, 0, 0, 0, 0, 0]])
@pytest.mark.parametrize("shape,kind,ns,maxd", [
    ((72, 60), sk.SyntheticKind.Fractal, 24, None),
    ((64, 80), sk.SyntheticKind.SmoothedNoise, 36, 200.0),
])
def test_devices_shared_gpu_sum_to_total(devices, shape, kind, ns, maxd):
    """Ranks sharing the GPU: each runs its row block of every sector into a
    private map, peer adds reduce them; raw and scaled maps within 1e-12 of
    the reference, over repeated calls while the cuts adapt."""
    dem = sk.make_synthetic(kind, *shape, 10.0, 9)
    cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=maxd, units=sk.Units.SquareKilometers)
    ora = _ora()
    ref_raw = ora.total_viewshed(dem.values, 10.0, ns, 1.5, max_distance=maxd or 0.0, raw=True)
    ref_vs = ora.total_viewshed(dem.values, 10.0, ns, 1.5, max_distance=maxd or 0.0, units=1)
    for _ in range(4):  # the first three calls move the cuts
        st = sk.EngineStats()
        raw = sk.total_viewshed_devices(dem, cfg, devices, raw=True, stats=st)
        np.testing.assert_allclose(raw, ref_raw, rtol=1e-12, atol=0)
        assert st.sectors == ns // 2 and st.kernel_launches > 0
        assert st.target_evals == sk.total_target_evals(ns, *shape, 10.0, maxd)
    vs = sk.total_viewshed_devices(dem, cfg, devices)
    np.testing.assert_allclose(vs, ref_vs, rtol=1e-12, atol=0)


@pytest.mark.gpu
def test_devices_errors():
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 20, 20, 10.0, 5)
    n = sk.device_count()
    with pytest.raises(ValueError, match="requested"):
        sk.total_viewshed_devices(dem, sk.RunConfig(ns=8), [0, n])
    with pytest.raises(ValueError, match="requested"):
        sk.total_viewshed(dem, sk.RunConfig(ns=8, n_gpus=n + 1))
    bad = dem.values.copy()
    bad[7, 11] = np.nan
    with pytest.raises(ValueError, match=r"non-finite elevation at cell \(7, 11\)"):
        sk.total_viewshed_devices(sk.Dem(bad, 10.0), sk.RunConfig(ns=8), [0, 0])
    with pytest.raises(ValueError, match="ns must be an even integer"):
        sk.total_viewshed_devices(dem, sk.RunConfig(ns=7), [0, 0])


@pytest.mark.gpu
def test_nccl_reduce_one_rank_bitexact():
    """The NCCL path itself (dlopen of libnccl, ncclCommInitAll, grouped
    ncclReduce on the ranks' streams) as a one-rank communicator, forced with
    SKS_NCCL=1 in a fresh process; bit-exact (a one-rank reduce is a copy)."""
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_2003_02200_b200 as sk
from _oracle import Ref, Orc, have_ref
dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 64, 56, 10.0, 3)
cfg = sk.RunConfig(ns=36, h0=1.5, units=sk.Units.SquareMeters)
ora = Ref() if have_ref() else Orc()
ref = ora.total_viewshed(dem.values, 10.0, 36, 1.5, raw=True)
st = sk.EngineStats()
ours = sk.total_viewshed_devices(dem, cfg, [0], raw=True, stats=st)
assert np.array_equal(ours.view(np.uint64), ref.view(np.uint64))
maps = open("/proc/self/maps").read()
assert "libnccl" in maps, "NCCL not loaded"
print("nccl ok", st.reduce_seconds)
""" % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, SKS_NCCL="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "nccl ok" in r.stdout


# ---- one process per GPU (torch.distributed), the bench's N > 1 path --------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rows_worker(rank, world, port, shape, ns, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2003_02200_b200 as sk
    from paper_2003_02200_b200.distributed import RowBalancer, total_viewshed_distributed

    torch.cuda.set_device(0)  # the ranks share the box's one GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, *shape, 10.0, 7).values
    cfg = sk.RunConfig(ns=ns, h0=1.5, units=sk.Units.SquareMeters)
    ctx = sk.Context(0)
    bal = RowBalancer(world)
    outs = []
    for _ in range(3):
        stats = {}
        res = total_viewshed_distributed(dem, 10.0, cfg, raw=True, context=ctx, stats=stats, mode="rows",
                                         cuts=bal.cuts)
        es = stats["rank_stats"]
        t = torch.tensor([es.skew_seconds + es.scan_seconds + es.fixup_seconds + es.unskew_seconds],
                         dtype=torch.float64)
        got = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(got, t)
        bal.update([float(x) for x in got])
        outs.append(res)
    q.put((rank, outs, bal.cuts.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_row_sharding_with_rebalancing():
    """World 2 over gloo on one B200 (NCCL refuses two ranks on one device):
    mode="rows" (every rank runs its row block of every sector), the
    RowBalancer moving the cuts between calls, one reduce of the f64 maps —
    the reduced map on rank 0 within 1e-12 of the reference every time."""
    import torch.multiprocessing as mp

    shape, ns = (96, 80), 36
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, *shape, 10.0, 7).values
    ref = _ora().total_viewshed(dem, 10.0, ns, 1.5, raw=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, shape, ns, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, outs, cuts = q.get(timeout=300)
        got[rank] = (outs, cuts)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs0, cuts0 = got[0]
    assert all(o is None for o in got[1][0])
    assert cuts0 == got[1][1]  # every rank computed the same cuts
    for o in outs0:
        np.testing.assert_allclose(o, ref, rtol=1e-12, atol=0)
