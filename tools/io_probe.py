"""BPST/BPVL I/O throughput: write and read back the BASELINE stack and a 512^3 volume
through the library (direct to pinned memory)."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp

d = sys.argv[1] if len(sys.argv) > 1 else "/tmp"
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
p = os.path.join(d, "probe.bpst")
t0 = time.perf_counter(); s.write(p); tw = time.perf_counter() - t0
nb = os.path.getsize(p)
for rep in range(2):
    t0 = time.perf_counter(); s2 = bp.Stack.read(p); tr = time.perf_counter() - t0
    print(f"stack {nb / 1e9:.2f} GB: write {nb / tw / 1e9:.2f} GB/s, read (page cache, rep {rep}) {nb / tr / 1e9:.2f} GB/s")
    s2.close()
v = bp.Volume.create(512)
pv = os.path.join(d, "probe.bpvl")
t0 = time.perf_counter(); v.write(pv); tw = time.perf_counter() - t0
nv = os.path.getsize(pv)
t0 = time.perf_counter(); v2 = bp.Volume.read(pv); tr = time.perf_counter() - t0
print(f"volume {nv / 1e9:.2f} GB: write {nv / tw / 1e9:.2f} GB/s, read {nv / tr / 1e9:.2f} GB/s")
os.remove(p); os.remove(pv)
