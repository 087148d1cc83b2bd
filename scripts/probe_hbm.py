"""Dev probe: device-to-device copy bandwidth (read + write bytes) vs buffer
size and duration, the same method as MEASURED_PEAKS.json's hbm_gbs."""
import torch
for gib in (0.25, 1, 2, 5, 10):
    n = int(gib * (1 << 30) // 2)  # bf16 elements per buffer
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    best, tot_t, tot_b = 0.0, 0.0, 0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, 4 * n / ms / 1e6)
    # sustained: back to back for ~1 s
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(3, int(1.0 / (4 * n / 6.4e12)))
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record(); torch.cuda.synchronize()
    sus = 4 * n * reps / e0.elapsed_time(e1) / 1e6
    print(f"{2 * gib:5.1f} GiB moved per copy: best {best:7.1f} GB/s, sustained {sus:7.1f} GB/s ({reps} copies)")
    del a, b
    torch.cuda.empty_cache()
