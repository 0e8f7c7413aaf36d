"""Does a PCIe H2D copy slow down while HBM-heavy kernels run? (experiment)"""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty(n, dtype=torch.int32, device="cuda")
a = torch.empty(1 << 29, dtype=torch.int32, device="cuda")
b = torch.empty(1 << 29, dtype=torch.int32, device="cuda")
cs = torch.cuda.Stream()
def h2d():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs); d.copy_(h, non_blocking=True); e1.record(cs)
    return e0, e1
for it in range(2):
    torch.cuda.synchronize()
    e0, e1 = h2d(); torch.cuda.synchronize(); print("H2D alone ms", e0.elapsed_time(e1))
    torch.cuda.synchronize()
    e0, e1 = h2d()
    k0 = torch.cuda.Event(enable_timing=True); k1 = torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(60): b.copy_(a)
    k1.record()
    torch.cuda.synchronize(); print("H2D with copies ms", e0.elapsed_time(e1), "copies ms", k0.elapsed_time(k1), "(alone ~", 60*4*2*(1<<29)/6.5e12*1e3, ")")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs); h.copy_(d, non_blocking=True); e1.record(cs)
    torch.cuda.synchronize(); print("D2H alone ms", e0.elapsed_time(e1))
