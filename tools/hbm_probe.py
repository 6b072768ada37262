"""HBM probe (dev tool): achieved bandwidth of plain torch write / copy / read streams of the
radio fp16 output size, to compare the fused kernel's store-heavy traffic with what a pure
stream reaches on this box.  Prints GB/s (bytes moved / time)."""
import torch

n = 2 * 1024 ** 3 // 4  # 2 GiB of fp32 (radio fp16 output = 2.15 GB)
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n // 4, dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e-3


s = t(lambda: a.fill_(1.0))
print(f"write-only fill 2 GiB: {a.numel() * 4 / s / 1e9:.0f} GB/s")
h = a[: n // 2]
s = t(lambda: h.copy_(a[n // 2:]))
print(f"copy 1 GiB -> 1 GiB: {a.numel() * 4 / s / 1e9:.0f} GB/s (read + write)")
s = t(lambda: a.sum())
print(f"read-only sum 2 GiB: {a.numel() * 4 / s / 1e9:.0f} GB/s")
# 1 : 4 read : write mix like the radio step (0.54 GB read, 2.15 GB written)
c = a[: n // 4 * 4].view(4, n // 4)
s = t(lambda: c.copy_(b.expand(4, n // 4)))
print(f"read 0.5 GiB broadcast into 2 GiB write: {(b.numel() + c.numel()) * 4 / s / 1e9:.0f} GB/s")
