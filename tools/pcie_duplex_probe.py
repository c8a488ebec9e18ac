"""PCIe copy bandwidth on the box: pinned H2D alone, D2H alone, and both at once on two
streams (is the link full duplex for this workload's sizes?).  2.38 GB H2D / 0.54 GB D2H,
the per-reconstruction traffic at 512^3, in 32 MB chunks."""
import torch, time
H, D, CH = 2376990720, 536870912, 32 << 20
h_src = torch.empty(H // 4, dtype=torch.float32).pin_memory()
d_dst = torch.empty(H // 4, dtype=torch.float32, device="cuda")
d_src = torch.empty(D // 4, dtype=torch.float32, device="cuda")
h_dst = torch.empty(D // 4, dtype=torch.float32).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def h2d():
    with torch.cuda.stream(s1):
        for o in range(0, H // 4, CH // 4):
            d_dst[o:o + CH // 4].copy_(h_src[o:o + CH // 4], non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        for o in range(0, D // 4, CH // 4):
            h_dst[o:o + CH // 4].copy_(d_src[o:o + CH // 4], non_blocking=True)
def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
for _ in range(2): timed(h2d); timed(d2h)
a = min(timed(h2d) for _ in range(3)); b = min(timed(d2h) for _ in range(3))
c = min(timed(lambda: (h2d(), d2h())) for _ in range(3))
print(f"H2D {H/1e9:.2f} GB: {a:.1f} ms ({H/a/1e6:.1f} GB/s); D2H {D/1e9:.2f} GB: {b:.1f} ms ({D/b/1e6:.1f} GB/s); "
      f"both concurrently: {c:.1f} ms (sum {a+b:.1f}, max {max(a,b):.1f}); combined {(H+D)/c/1e6:.1f} GB/s")
