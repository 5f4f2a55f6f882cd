"""Write-only and read-only HBM bandwidth of this B200 (the conv1 / conv3 rooflines): memset / fill of 2.15 GB (h1's
size) and a sum over 1.07 GB (h2's size), CUDA events, best of 10."""
import json, torch
def best(fn, k=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
h1 = torch.empty(2 * 4096 * 4096 * 64 // 2, dtype=torch.bfloat16, device="cuda")   # 2.15 GB
h2 = torch.empty(4096 * 4096 * 32, dtype=torch.bfloat16, device="cuda").normal_()  # 1.07 GB
dst = torch.empty_like(h2)
out = {}
t = best(lambda: h1.zero_()); out["memset_2.15GB_ms"] = t; out["write_GBs"] = h1.numel() * 2 / t / 1e6
t = best(lambda: h1.fill_(1.0)); out["fill_GBs"] = h1.numel() * 2 / t / 1e6
t = best(lambda: h2.sum(dtype=torch.float32)); out["read_sum_GBs"] = h2.numel() * 2 / t / 1e6
t = best(lambda: dst.copy_(h2)); out["copy_rw_GBs"] = 2 * h2.numel() * 2 / t / 1e6
print(json.dumps({k: round(v, 3) for k, v in out.items()}))
