"""HBM write-only and read-only bandwidth on this GPU (torch fill_ / sum over 2 GiB, CUDA events):
the roofline of output-bound layers (conv1_1, the ResNet stem, 1x1 expansions)."""
import torch
n = 1 << 30  # bf16 elements = 2 GiB
x = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in [("write (fill_)", lambda: x.fill_(1.0), 2 * n), ("write (zero_)", lambda: x.zero_(), 2 * n),
                         ("read (sum)", lambda: x.sum(dtype=torch.float32), 2 * n),
                         ("copy (read+write)", lambda: y.copy_(x), 4 * n)]:
    if name.startswith("copy"):
        y = torch.empty_like(x)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"{name:20s} {nbytes / best / 1e6:8.1f} GB/s")
