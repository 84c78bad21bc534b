"""Probe: device write-only and read-only streaming bandwidth (torch fill_ / sum over 512 MiB),
to bound adv-norm phase C (adv_tok writes) and phase A (mask reads).  Plumbing only."""
import torch

n = 128 << 20  # floats (512 MiB)
x = torch.empty(n, dtype=torch.float32, device="cuda")
m = torch.empty(n, dtype=torch.uint8, device="cuda")
m.fill_(1)
for name, fn, nbytes in (("write fill_ f32 512 MiB", lambda: x.fill_(1.0), 4 * n),
                         ("read u8 sum 128 MiB", lambda: m.sum(dtype=torch.int32), n),
                         ("copy f32 256 MiB -> 256 MiB", lambda: x[: n // 2].copy_(x[n // 2:]), 4 * n)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {best * 1e3:.1f} us, {nbytes / best / 1e6:.0f} GB/s", flush=True)
