"""Time the GPU FDK filter alone on full-size views (resident), for ncu / A-B."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1104_5243_b200 as bp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rng = np.random.default_rng(1)
px = rng.uniform(0, 1, size=(n, 960, 1248)).astype(np.float32)
bp.filter_views(px[:2], 750.0, 1200.0, 0.32)
t0 = time.perf_counter()
bp.filter_views(px, 750.0, 1200.0, 0.32)
dt = time.perf_counter() - t0
print(f"filter_views {n} views incl. H2D/D2H: {dt*1e3:.1f} ms ({dt*1e3/n:.3f} ms/view)")
