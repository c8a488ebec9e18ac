"""Throughput of back-to-back streamed reconstructions through the module C ABI with NC
contexts on NC host threads (default 2) (double-buffered: one volume's readback overlaps the next
volume's upload).  Every reconstruction uploads its whole pinned stack and reads its whole
volume back inside the timed window.  Env: AB_L (512), AB_BATCH (32), AB_STEPS (6)."""
import os, sys, threading, time
sys.path.insert(0, ".")
import numpy as np
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512"))
B = int(os.environ.get("AB_BATCH", "32"))
K = int(os.environ.get("AB_STEPS", "6"))
NC = int(os.environ.get("AB_CTX", "2"))
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
vols = [bp.Volume.create(L) for _ in range(NC)]
RB = int(os.environ.get("AB_RING", "0"))
ctxs = [bp.GpuContext(L, 1248, 960, device=0, strict=False, view_batch=B, ring_batches=RB) for _ in range(NC)]
for c, v in zip(ctxs, vols):  # warm-up
    c.backproject_stack(s)
    c.finish(out=v.data)
ref = vols[0].data.copy()
go = threading.Barrier(NC + 1)
def worker(i, n):
    go.wait()
    for _ in range(n):
        ctxs[i].backproject_stack(s)
        ctxs[i].finish(out=vols[i].data)
ts = [threading.Thread(target=worker, args=(i, K // NC + (1 if i < K % NC else 0))) for i in range(NC)]
for t in ts: t.start()
go.wait()
t0 = time.perf_counter()
for t in ts: t.join()
dt = time.perf_counter() - t0
same = all(np.array_equal(v.data.view(np.int32), ref.view(np.int32)) for v in vols)
print(f"pipelined e2e L={L} B={B} contexts={NC}: {K} reconstructions in {dt * 1e3:.1f} ms -> {dt * 1e3 / K:.2f} ms each, "
      f"{K * 496 * L ** 3 / dt / 1e9:.1f} GUP/s; volumes bitwise equal to the sequential run: {same}")
for c in ctxs: c.close()
