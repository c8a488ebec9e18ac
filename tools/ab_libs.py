"""Compile-time A/B of library builds: resident 512^3 timing plus an accuracy check.

Usage: python tools/ab_libs.py name=path.so [name=path.so ...]
Each build runs in its own process (BP_LIB_PATH), rounds interleaved (ABCABC...).
The first round of each build also saves sampled lines of its fast-mode volume;
every build is compared with the first one (max / RMS of the difference relative to
max|first| over the sample).  Env: AB_L (512), AB_BATCH (248), AB_ROUNDS (3), AB_REPS (3),
AB_STRICT (0), AB_ARCP (0).
"""
import json
import os
import statistics
import subprocess
import sys

import numpy as np

CHILD = r"""
import os, sys, json, numpy as np
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512")); B = int(os.environ.get("AB_BATCH", "248"))
reps = int(os.environ.get("AB_REPS", "3"))
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
with bp.GpuContext(L, 1248, 960, device=0, strict=os.environ.get("AB_STRICT") == "1",
                   view_batch=B, ring_batches=(496 + B - 1) // B, profile_launches=True,
                   recip_mode=3 if os.environ.get("AB_ARCP") == "1" else 0) as c:
    c.upload_stack(s)
    c.time_resident(1)
    v, kv = [], []
    for _ in range(reps):
        ms, st = c.time_resident(1)
        v.append(ms); kv.append(st.kernel_ms)
    out = os.environ.get("AB_LINES")
    if out:
        rng = np.random.default_rng(7)
        ys = rng.integers(0, L, 2048); zs = rng.integers(0, L, 2048)
        np.save(out, c.read_lines(ys, zs))
print(json.dumps({"ms": v, "kernel_ms": kv, "tile": [st.tile_w, st.tile_h],
                  "fallback": st.fallback_pairs}))
"""


def main():
    builds = [a.split("=", 1) for a in sys.argv[1:]]
    rounds = int(os.environ.get("AB_ROUNDS", "3"))
    L = int(os.environ.get("AB_L", "512"))
    res = {n: [] for n, _ in builds}
    kres = {n: [] for n, _ in builds}
    for r in range(rounds):
        for name, path in builds:
            env = dict(os.environ, BP_LIB_PATH=os.path.abspath(path))
            if r == 0:
                env["AB_LINES"] = f"/tmp/ab_lines_{name}.npy"
            p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True,
                               text=True)
            if p.returncode != 0:
                print(f"{name}: FAILED rc={p.returncode}\n{p.stderr[-2000:]}")
                continue
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res[name] += d["ms"]
            kres[name] += d["kernel_ms"]
    first = builds[0][0]
    ref = np.load(f"/tmp/ab_lines_{first}.npy").astype(np.float64)
    peak = np.abs(ref).max()
    for name, _ in builds:
        if not res[name]:
            continue
        med = statistics.median(res[name])
        kmed = statistics.median(kres[name])
        acc = ""
        if name != first and os.path.exists(f"/tmp/ab_lines_{name}.npy"):
            d = np.load(f"/tmp/ab_lines_{name}.npy").astype(np.float64) - ref
            acc = (f" | vs {first}: max {np.abs(d).max() / peak:.2e} rms "
                   f"{np.sqrt((d * d).mean()) / peak:.2e} of max|{first}|")
        print(f"{name:10s} L={L} median {med:.2f} ms (kernels {kmed:.2f}) -> "
              f"{496 * L ** 3 / med / 1e6:.1f} GUP/s  all {[round(x, 2) for x in res[name]]}{acc}")


if __name__ == "__main__":
    main()
