"""Read-bandwidth reference points for the scorer sweep's 512 MiB
(development aid): torch reductions / copy over the same bytes, L2 flushed."""
import torch
B, G = 4096, 16384
x = torch.randint(0, 1 << 30, (B, G), device="cuda", dtype=torch.int64)
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, bytes_):
    ts = []
    for i in range(8):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    m = sorted(ts[2:])[len(ts[2:]) // 2]
    return f"{m*1e3:.1f} us {bytes_/m/1e6:.0f} GB/s"
nb = x.numel() * 8
print("sum   ", t(lambda: x.sum(), nb))
print("amax  ", t(lambda: x.amax(), nb))
print("copy  ", t(lambda: y.copy_(x), 2 * nb))
xs = x[:, :4096].contiguous()
print("sum 128MiB", t(lambda: xs.sum(), xs.numel() * 8))
x2 = torch.randint(0, 1 << 30, (4 * B, G), device="cuda", dtype=torch.int64)
print("sum 2GiB", t(lambda: x2.sum(), x2.numel() * 8))
