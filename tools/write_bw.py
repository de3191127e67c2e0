"""HBM write-only and copy bandwidth on this GPU (torch fill / copy kernels,
CUDA events, best of 10): the roofline of a write-bound kernel such as the
relocation (8N sDEM + cv-zero writes, DEM reads from L2)."""
import json
import torch

n = 3 << 30  # bytes
a = torch.empty(n // 4, dtype=torch.int32, device="cuda")
b = torch.empty(n // 4, dtype=torch.int32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        t.append(ev[0].elapsed_time(ev[1]) / 1e3)
    return min(t)


res = {
    "write_zero_gbs": n / best(lambda: a.zero_()) / 1e9,
    "write_fill_gbs": n / best(lambda: a.fill_(7)) / 1e9,
    "memset_gbs": n / best(lambda: torch.cuda.current_stream() and a.data.zero_()) / 1e9,
    "copy_rw_gbs": 2 * n / best(lambda: b.copy_(a)) / 1e9,
    "read_sum_gbs": n / best(lambda: a.sum()) / 1e9,
}
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
