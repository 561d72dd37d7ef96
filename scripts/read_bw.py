"""Read-only HBM bandwidth probe (torch reductions over an 8 GiB buffer)."""
import torch
x = torch.ones(2 ** 31, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
for name, fn in (("sum_int32", lambda: x.sum()), ("amax_int32", lambda: x.amax()),
                 ("copy", lambda: y.copy_(x[: 2 ** 30]))):
    if name == "copy":
        y = torch.empty(2 ** 30, dtype=torch.int32, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = x.numel() * 4 if name != "copy" else 2 * y.numel() * 4
    print(f"{name}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
