"""A/B timing harness: one process, one stack, configs interleaved (ABAB...)."""
import os, sys, statistics
sys.path.insert(0, ".")
import paper_1104_5243_b200 as bp
L = int(os.environ.get("AB_L", "512"))
configs = [c.split("=", 1) if "=" in c else (c, "") for c in sys.argv[1:]]  # ENV=VAL or label
s = bp.Stack.baseline(n_views=496, isx=1248, isy=960)
res = {}
def env_apply(spec):
    for kv in spec.split(","):
        if not kv: continue
        k, v = kv.split(":")
        if v == "-": os.environ.pop(k, None)
        else: os.environ[k] = v
for rnd in range(3):
    for spec in sys.argv[1:]:
        env_apply(spec)
        with bp.GpuContext(L, 1248, 960, device=0, strict=os.environ.get("AB_STRICT") == "1",
                           view_batch=32, ring_batches=16) as c:
            c.upload_stack(s)
            c.time_resident(1)
            for _ in range(3):
                ms, st = c.time_resident(1)
                res.setdefault(spec, []).append(ms)
        # reset env to defaults for next spec
        for kv in spec.split(","):
            if kv: os.environ.pop(kv.split(":")[0], None)
for spec, v in res.items():
    med = statistics.median(v)
    print(f"{spec:40s} median {med:.2f} ms  min {min(v):.2f}  -> {496 * L**3 / med / 1e6:.1f} GUP/s nominal")
