"""PCIe H2D / D2H throughput probe (pinned host memory), to size the e2e bound."""
import time
import torch

n = 2377121792 // 4  # the BASELINE stack, floats
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")


def run(chunk_mb, nstreams):
    ch = chunk_mb * (1 << 20) // 4
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, off in enumerate(range(0, n, ch)):
        with torch.cuda.stream(streams[i % nstreams]):
            d[off:off + ch].copy_(h[off:off + ch], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return n * 4 / dt / 1e9


def run_d2h(chunk_mb, nstreams):
    m = 536870912 // 4
    ch = chunk_mb * (1 << 20) // 4
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, off in enumerate(range(0, m, ch)):
        with torch.cuda.stream(streams[i % nstreams]):
            h[off:off + ch].copy_(d[off:off + ch], non_blocking=True)
    torch.cuda.synchronize()
    return m * 4 / (time.perf_counter() - t0) / 1e9


for rep in range(2):
    for mb, s in [(4, 1), (4, 2), (4, 4), (16, 1), (16, 2), (64, 1), (64, 2)]:
        print(f"H2D chunk {mb} MB streams {s}: {run(mb, s):.1f} GB/s")
    for mb, s in [(4, 1), (16, 2), (64, 1)]:
        print(f"D2H chunk {mb} MB streams {s}: {run_d2h(mb, s):.1f} GB/s")
