#!/usr/bin/env python3
"""Benchmark: GUP/s of the 512^3 x 496-view voxel-driven FDK backprojection
(BASELINE.json metric, config 3) on B200, next to the reference CPU path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--l 512]

A "step" = one complete reconstruction (all 496 views) of the L^3 volume.
  value      : nominal GUP/s (views * L^3 / s) with the projections resident in HBM,
               CUDA-event time on the library's compute stream, max over ranks.
  e2e        : the same metric through the public C ABI streaming call
               (bp_gpu_backproject_async from pinned host memory + bp_gpu_finish into a
               pinned host volume): H2D of every view and D2H of the volume are inside
               the timed region.  Host wall clock around the API calls.
  roofline   : binding roofline of the dominant kernel = shared-memory load bandwidth
               (16 B of texel loads per VISIBLE voxel update).
  cpu_baseline: the reference's own bp::reconstruct (oracle/_ref, built from
               /root/reference sources) on a bounded sample of the workload.
Inputs are seeded synthetic (BASELINE.json configs).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "GUP/s (voxel updates/s) for 512^3x496-view backprojection"
SMEM_BYTES_PER_SM_CLK = 128.0
CONFIG_OF_L = {128: 1, 256: 2, 512: 3, 1024: 4, 2048: 5}
N_SM = 148


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names[1:], p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_stack(args):
    import paper_1104_5243_b200 as bp
    t0 = time.time()
    s = bp.Stack.baseline(n_views=args.views, isx=1248, isy=960, seed=args.seed)
    return s, time.time() - t0


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation (oracle/_ref: the unmodified
# reference sources, compiled by oracle/Makefile), driven through ITS public C ABI
# (bp_stack_read + bp_reconstruct, proj/include/backproject.h).  The process never
# loads this repository's library: the seeded BASELINE stack is written to a BPST file
# by a separate process (`bench.py --write-stack`), and the reference's own reader
# loads it.

class RefReconParams(ctypes.Structure):
    """bp_recon_params, proj/include/backproject.h:60-73."""
    _fields_ = [("l", ctypes.c_uint32), ("threads", ctypes.c_int), ("chunk", ctypes.c_int),
                ("block_b", ctypes.c_int), ("lanes", ctypes.c_int), ("recip_mode", ctypes.c_int),
                ("extract", ctypes.c_int), ("strict_mode", ctypes.c_int),
                ("distance_weight", ctypes.c_int), ("clip", ctypes.c_int),
                ("numa_domains", ctypes.c_int), ("clip_cache", ctypes.c_char_p)]


class RefReconStats(ctypes.Structure):
    """bp_recon_stats, proj/include/backproject.h:75-84."""
    _fields_ = [("seconds", ctypes.c_double), ("voxel_updates", ctypes.c_uint64),
                ("gups", ctypes.c_double), ("gflops", ctypes.c_double),
                ("writeback_stores", ctypes.c_uint64), ("bytes_copied", ctypes.c_uint64),
                ("clip_reduction", ctypes.c_double), ("thread_updates_min", ctypes.c_uint64),
                ("thread_updates_max", ctypes.c_uint64)]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def stack_file(views: int, seed: int, sample: int) -> str:
    """BPST file of the first `sample` views of the seeded `views`-view BASELINE stack,
    written by a separate process (this process must not load the repo's library)."""
    d = os.environ.get("BP_BENCH_TMP", "/tmp")
    path = os.path.join(d, f"bp_baseline_s{seed}_v{views}_n{sample}.bpst")
    want = 16 + sample * (96 + 4 * 1248 * 960)  # BPST: magic, isx, isy, count, matrices, pixels
    if not (os.path.exists(path) and os.path.getsize(path) >= want):
        subprocess.run([sys.executable, os.path.abspath(__file__), "--write-stack", path,
                        "--views", str(views), "--seed", str(seed), "--sample-views", str(sample)],
                       check=True)
    return path


def write_stack(args):
    import paper_1104_5243_b200 as bp
    s = bp.Stack.baseline(n_views=args.views, isx=1248, isy=960, seed=args.seed)
    n = args.sample_views or args.views
    if n < args.views:
        s = bp.Stack.from_arrays(s.pixels[:n], s.matrices[:n])
    tmp = args.write_stack + ".part"
    s.write(tmp)
    os.replace(tmp, args.write_stack)
    return 0


def reference_reconstructions(path, L, steps, warmup, threads):
    """Times `steps` complete bp_reconstruct calls of the reference (lanes 8, block_b 8,
    clip on with its own clip_cache, exact reciprocal: BASELINE.md section 3) on the BPST
    stack at `path`.  Returns (per-step wall seconds, last stats, views)."""
    from oracle import oracle as O  # ctypes loader of oracle/_ref only
    R = O.ref()
    if R is None:
        raise RuntimeError("oracle/_ref (the reference library) is not built")
    R.bp_stack_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    R.bp_stack_dims.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32),
                                ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
    R.bp_stack_free.argtypes = [ctypes.c_void_p]
    R.bp_reconstruct.argtypes = [ctypes.c_void_p, ctypes.POINTER(RefReconParams),
                                 ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(RefReconStats)]
    R.bp_volume_free.argtypes = [ctypes.c_void_p]
    R.bp_last_error.restype = ctypes.c_char_p
    h = ctypes.c_void_p()
    if R.bp_stack_read(path.encode(), ctypes.byref(h)) != 0:
        raise RuntimeError(R.bp_last_error().decode())
    isx, isy, cnt = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    R.bp_stack_dims(h, ctypes.byref(isx), ctypes.byref(isy), ctypes.byref(cnt))
    cache = path + f".L{L}.bpct"
    p = RefReconParams(l=L, threads=threads, chunk=1, block_b=8, lanes=8, recip_mode=0, extract=0,
                       strict_mode=1, distance_weight=1, clip=1, numa_domains=1,
                       clip_cache=cache.encode())
    walls, st = [], RefReconStats()
    for i in range(warmup + steps):
        vol = ctypes.c_void_p()
        t0 = time.perf_counter()
        rc = R.bp_reconstruct(h, ctypes.byref(p), ctypes.byref(vol), ctypes.byref(st))
        dt = time.perf_counter() - t0
        if rc != 0:
            raise RuntimeError(R.bp_last_error().decode())
        R.bp_volume_free(vol)
        if i >= warmup:
            walls.append(dt)
    R.bp_stack_free(h)
    return walls, st, int(cnt.value)


def run_reference_arm(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    L = args.l
    threads = os.cpu_count() or 1
    # bounded: one full reconstruction writes the reference's clip cache (untimed), then
    # at most --ref-steps complete 496-view reconstructions are timed (about a minute each
    # on 16 cores), whatever --steps asks for, so the arm ends within a few minutes
    steps = max(1, min(args.steps, args.ref_steps))
    warmup = 1 if args.warmup > 0 else 0
    t0 = time.time()
    sample = args.ref_sample_views or args.views
    path = stack_file(args.views, args.seed, sample)
    prep_s = time.time() - t0
    walls, st, n = reference_reconstructions(path, L, steps, warmup, threads)
    wall = float(np.median(walls))
    nominal = n * L ** 3
    v = nominal / wall / 1e9
    line = {
        "metric": METRIC, "value": v, "unit": "GUP/s", "n_gpus": args.gpus, "steps": steps,
        "steps_requested": args.steps, "warmup": warmup, "ms_per_step": wall * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{L}^3 x {n} views of 1248x960" + (
                       f" (BASELINE config {CONFIG_OF_L[L]})" if L in CONFIG_OF_L and n == 496 else ""),
                   "l": L, "views": n, "api": "reference bp_stack_read + bp_reconstruct (oracle/_ref, "
                                      "unmodified reference sources)",
                   "params": "threads=all lanes=8 block_b=8 clip=1 (reference clip_cache) "
                             "recip=exact distance_weight=1"},
        "cpu_baseline": {"value": v, "unit": "GUP/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": (f"all {n} views" if n == args.views else
                                    f"the first {n} of {args.views} views") +
                                   f", full {L}^3 volume, {steps} timed bp_reconstruct call(s) after "
                                   f"{warmup} untimed one (median wall time per call)"},
        "e2e": {"value": v, "unit": "GUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_stats": {"timed_region_s": st.seconds, "voxel_updates": int(st.voxel_updates),
                            "gups_performed": st.gups, "clip_reduction": st.clip_reduction,
                            "walls_s": walls},
        "stack_prep_s": prep_s,
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_subprocess(args, sample):
    """The reference arm's code on the first `sample` views, in a child process (so this
    process's GPU library stays out of the reference's way)."""
    stack_file(args.views, args.seed, sample)
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--steps", "1",
           "--warmup", "1", "--views", str(args.views), "--seed", str(args.seed), "--l", str(args.l),
           "--ref-sample-views", str(sample)]
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if p.returncode != 0:
        return None
    return json.loads(p.stdout.strip().splitlines()[-1])


# ---------------------------------------------------------------------------
# our arm

def _load_profile_summary():
    try:
        with open(os.path.join(ROOT, "profiles", "latest.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def run_ours(args):
    import paper_1104_5243_b200 as bp
    rank, world, local = dist_env()
    dist = torch = None
    ctrl = "cuda"  # device of the control-plane tensors (max-reduce of timings etc.)
    if world > 1:
        import torch
        import torch.distributed as dist  # plumbing: barrier, max-reduce, slab gather
        torch.cuda.set_device(local % torch.cuda.device_count())
        # BP_BENCH_BACKEND=gloo runs the control plane on CPU tensors: it lets the
        # multi-rank flow (slabs, row windows, fused IPC gather) be exercised with
        # several ranks on ONE GPU -- correctness only, never a scaling number
        backend = os.environ.get("BP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            dist.init_process_group(backend)
            ctrl = "cpu"
    n_dev = bp.device_count()
    if n_dev < 1:
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        return 1
    device = local % n_dev
    L = args.l
    stack, gen_s = make_stack(args)
    px, mats = stack.pixels, stack.matrices
    n, isy, isx = px.shape

    # slab of this rank (work-balanced partition, identical on every rank)
    if world > 1:
        bounds = bp.partition_slabs(mats, isx, isy, L, world)
        z0, z1 = int(bounds[rank]), int(bounds[rank + 1])
    else:
        bounds = [0, L]
        z0, z1 = 0, L

    # ---- visible updates (clip_stats semantics) for the roofline -------------
    with bp.GpuContext(L, isx, isy, device=device, z_begin=z0, z_end=z1, count_visible=True,
                       view_batch=32) as c:
        c.backproject_stack(stack)
        _, vst = c.finish(readback=False)
    visible = int(vst.visible_updates)

    # ---- value: resident projections, device-event timing ---------------------
    ring = (n + args.batch - 1) // args.batch
    slab_t = full_t = None
    out_ptr = None  # fused gather: the final pass of each rank stores into rank 0's volume
    fused = False
    if world > 1:
        # The one exchange step is the slab gather to rank 0. It is fused into the last
        # kernel of every reconstruction: rank 0 exports its full volume through CUDA IPC,
        # and each rank's final pass stores its slab straight into it over NVLink. If
        # mapping fails on any rank, every rank falls back to an NCCL send/recv gather.
        if rank == 0:
            full_t = torch.empty((L, L, L), dtype=torch.float32, device="cuda")
        obj = [bp.ipc_handle(full_t.data_ptr()) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        base = None
        try:
            base = full_t.data_ptr() if rank == 0 else bp.ipc_open(obj[0])
            ok = 1
        except Exception:
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=ctrl)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        fused = int(flag.item()) == 1
        if fused:
            out_ptr = base + 4 * z0 * L * L
            slab_t = torch.empty((z1 - z0, L, L), dtype=torch.float32, device="cuda")
        else:
            if base is not None and rank != 0:
                bp.ipc_close(base)
            # rank 0's slab is a view into the full volume (no extra copy)
            slab_t = full_t[z0:z1] if rank == 0 else torch.empty((z1 - z0, L, L), dtype=torch.float32,
                                                                   device="cuda")
    ctx = bp.GpuContext(L, isx, isy, device=device, z_begin=z0, z_end=z1, strict=args.strict,
                        view_batch=args.batch, ring_batches=ring, profile_launches=True,
                        device_volume=slab_t.data_ptr() if slab_t is not None else None,
                        output_volume=out_ptr)
    ctx.upload_stack(stack)

    def gather_ms():
        """NCCL fallback of the exchange step: variable-size slabs to rank 0."""
        if world == 1 or fused:
            return 0.0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if rank == 0:
            for src in range(1, world):
                dist.recv(full_t[int(bounds[src]):int(bounds[src + 1])], src=src)
        else:
            dist.send(slab_t, dst=0)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        ctx.time_resident(1)
        gather_ms()
    if dist:
        dist.barrier()
    clk = ClockSampler(device)
    clk.start()
    ms = 0.0
    launches = 0
    prep_launches = 0
    kernel_ms = 0.0
    st = None
    for _ in range(args.steps):
        m, st = ctx.time_resident(1)
        ms += m + gather_ms()
        launches += int(st.launches)
        prep_launches += int(st.prep_launches)
        kernel_ms += float(st.kernel_ms)
    clocks = clk.stop()
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=ctrl)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        t = torch.tensor([launches + prep_launches], dtype=torch.float64, device=ctrl)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_launches = int(t.item())
    else:
        total_launches = launches + prep_launches
    nominal_step = n * L ** 3  # whole job, all ranks
    value = nominal_step * args.steps / (ms / 1e3) / 1e9
    per_launch_s = kernel_ms / 1e3 / max(1, launches)
    launches_per_step = launches / args.steps
    ctx.close()
    gather_check = None
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()  # all final-pass stores into rank 0's volume have landed
        if fused and rank != 0:
            bp.ipc_close(base)
        if args.verify_gather and rank == 0:
            # the gathered volume must equal a single-context reconstruction bitwise
            # (per-voxel arithmetic and view order do not depend on the slab split)
            one = torch.empty((L, L, L), dtype=torch.float32, device="cuda")
            vc = bp.GpuContext(L, isx, isy, device=device, strict=args.strict, view_batch=args.batch,
                               ring_batches=ring, device_volume=one.data_ptr())
            vc.upload_stack(stack)
            vc.time_resident(1)
            vc.close()
            torch.cuda.synchronize()
            gather_check = bool(torch.equal(one.view(torch.int32), full_t.view(torch.int32)))
            del one

    # strict (bitwise-reference) arithmetic on the same resident data, reported beside,
    # and the opt-in hardware-reciprocal tier (BP_RECIP_HW_APPROX) for the trade-off
    strict_ms = hwr_ms = None
    if not args.strict and world == 1:
        sctx = bp.GpuContext(L, isx, isy, device=device, strict=True, view_batch=args.batch,
                             ring_batches=ring)
        sctx.upload_stack(stack)
        sctx.time_resident(1)
        strict_ms, _ = sctx.time_resident(args.steps)
        sctx.close()
        hctx = bp.GpuContext(L, isx, isy, device=device, strict=False, view_batch=args.batch,
                             ring_batches=ring, recip_mode=bp.BP_RECIP_HW_APPROX)
        hctx.upload_stack(stack)
        hctx.time_resident(1)
        hwr_ms, _ = hctx.time_resident(args.steps)
        hctx.close()

    # ---- e2e: streamed through the C ABI from pinned host memory ---------------
    # views=n: the caller knows its view count (a RabbitCT-style harness does), so the
    # library uploads the last ~112 views band-ordered and reads z-chunks back under the
    # remaining upload (bp_gpu_config.views)
    e2e_ctx = bp.GpuContext(L, isx, isy, device=device, z_begin=z0, z_end=z1,
                            strict=args.strict, view_batch=args.e2e_batch, views=n)
    host_vol = bp.Volume.create(L)  # pinned (library pool); each rank reads back its slab
    out = host_vol.data[z0:z1]
    for _ in range(max(1, args.warmup)):
        e2e_ctx.backproject_stack(stack)
        e2e_ctx.finish(out=out)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    h2d = d2h = 0
    h2d_ms = d2h_ms = 0.0
    e2e_each = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        e2e_ctx.backproject_stack(stack)
        _, est = e2e_ctx.finish(out=out)
        e2e_each.append((time.perf_counter() - t1) * 1e3)
        h2d += est.h2d_bytes
        d2h += est.d2h_bytes
        h2d_ms += est.h2d_ms
        d2h_ms += est.d2h_ms
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s, h2d, d2h], dtype=torch.float64, device=ctrl)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        e2e_s, h2d, d2h = float(mx[0].item()), int(t[1].item()), int(t[2].item())
    e2e_ctx.close()
    e2e_val = nominal_step * args.steps / e2e_s / 1e9

    # ---- e2e_copy: the module path a RabbitCT-style harness uses -- bp_gpu_backproject
    # (copy semantics: the image is staged before the call returns, so the caller may
    # reuse its buffer) from ordinary PAGEABLE per-view buffers into a PAGEABLE host
    # volume ------------------------------------------------
    e2e_copy = None
    if world == 1 and not args.no_copy_path:
        pg_px = np.array(px, copy=True)  # pageable (numpy heap), not the library's pinned pool
        pg_vol = np.empty((L, L, L), np.float32)
        pg_vol.fill(0.0)
        cctx = bp.GpuContext(L, isx, isy, device=device, strict=args.strict, view_batch=args.e2e_batch,
                             views=n)
        for _ in range(max(1, min(2, args.warmup))):
            for k in range(n):
                cctx.backproject(pg_px[k], mats[k], copy=True)
            cctx.finish(out=pg_vol)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for k in range(n):
                cctx.backproject(pg_px[k], mats[k], copy=True)
            cctx.finish(out=pg_vol)
        copy_s = time.perf_counter() - t0
        cctx.close()
        e2e_copy = {"value": nominal_step * args.steps / copy_s / 1e9, "unit": "GUP/s",
                    "ms_per_step": copy_s * 1e3 / args.steps,
                    "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                    "note": "bp_gpu_backproject (copy semantics) per view from pageable buffers, "
                            "bp_gpu_finish into a pageable volume; staging and readback copies "
                            "on the library's host copy pool"}
        del pg_px, pg_vol

    # ---- e2e, back-to-back reconstructions: two module contexts on two host threads, so
    # one volume's readback (D2H) overlaps the next volume's upload (H2D) -- PCIe is full
    # duplex (tools/pcie_duplex_probe.py).  Every reconstruction still uploads its whole
    # pinned stack and reads its whole volume back inside the window -------------------
    e2e_pipe = None
    if world == 1 and not args.no_pipelined:
        import threading
        pvols = [host_vol, bp.Volume.create(L)]
        pctx = [bp.GpuContext(L, isx, isy, device=device, strict=args.strict,
                              view_batch=args.e2e_batch, tail_batches=0) for _ in range(2)]
        for c, v in zip(pctx, pvols):
            for _ in range(max(1, args.warmup)):
                c.backproject_stack(stack)
                c.finish(out=v.data)
        go = threading.Barrier(3)
        # an even count (both contexts equally busy), at least 12: the pipeline's fill
        # (both first uploads share the link) and drain are amortised
        nsteps = max(12, args.steps + (args.steps & 1))

        def worker(i, cnt):
            go.wait()
            for _ in range(cnt):
                pctx[i].backproject_stack(stack)
                pctx[i].finish(out=pvols[i].data)

        ths = [threading.Thread(target=worker, args=(i, nsteps // 2 + (i < nsteps % 2))) for i in range(2)]
        for t in ths:
            t.start()
        go.wait()
        t0 = time.perf_counter()
        for t in ths:
            t.join()
        pipe_s = time.perf_counter() - t0
        for c in pctx:
            c.close()
        e2e_pipe = {"value": nominal_step * nsteps / pipe_s / 1e9, "unit": "GUP/s",
                    "ms_per_step": pipe_s * 1e3 / nsteps, "steps": nsteps,
                    "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                    "note": "back-to-back reconstructions through two bp_gpu contexts on two host threads "
                            "(tail_batches 0): one volume's D2H overlaps the next volume's H2D; `e2e` is "
                            "one reconstruction at a time"}

    # ---- FDK e2e: the same stream with the GPU cosine + ramp
    # filter applied to every view in the ring before backprojection ----------------
    fdk = None
    if world == 1 and not args.no_fdk:
        geom = (750.0, 1200.0, 0.32 * 1248.0 / isx)
        fctx = bp.GpuContext(L, isx, isy, device=device, strict=args.strict,
                             view_batch=args.e2e_batch, filter=geom, views=n)
        for _ in range(max(1, args.warmup)):
            fctx.backproject_stack(stack)
            fctx.finish(out=out)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            fctx.backproject_stack(stack)
            fctx.finish(out=out)
        fdk_s = time.perf_counter() - t0
        fctx.close()
        fdk = {"value": nominal_step * args.steps / fdk_s / 1e9, "unit": "GUP/s",
               "ms_per_step": fdk_s * 1e3 / args.steps,
               "note": "e2e with GPU FDK preprocessing (cosine weight + Ram-Lak FFT filter, "
                       "bp_filter.cu) of each uploaded view; the reference has no filter"}

    # ---- CPU baseline (rank 0, N=1 only): the reference arm's code on a bounded sample
    # (the first --cpu-views views, full volume), in a child process ----------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_baseline_subprocess(args, args.cpu_views)
        if r is not None:
            cb = r["cpu_baseline"]
            cpu = {"value": r["value"], "unit": "GUP/s", "cores": cb["cores"], "kind": cb["kind"],
                   "cpu_model": cb.get("cpu_model"),
                   "sample": cb["sample"] + " (bp::reconstruct lanes=8 block_b=8 clip=1, "
                             "reference clip_cache)"}

    if dist:
        vt = torch.tensor([visible], dtype=torch.float64, device=ctrl)
        dist.all_reduce(vt, op=dist.ReduceOp.SUM)
        visible_all = int(vt.item())
    else:
        visible_all = visible
    if rank != 0:
        dist.destroy_process_group()
        return 0
    peaks = load_peaks()
    prof = _load_profile_summary()
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    sm_max = clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    # dominant kernel: tiled backprojection.  Algorithmic SMEM-load bytes per launch =
    # 16 B x visible updates per launch (4 fp32 texels per update).
    achieved = 16.0 * (visible / max(1e-9, launches_per_step)) / per_launch_s / 1e9
    tex_bytes = 4.0 if args.strict else 8.0  # bytes per detector texel the kernel reads
    peak_nominal = SMEM_BYTES_PER_SM_CLK * N_SM * float(sm_max) * 1e6 / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GUP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{L}^3 x {n} views of 1248x960 (BASELINE config 3)", "l": L,
                   "views": n, "view_batch": args.batch, "e2e_view_batch": args.e2e_batch,
                   "arithmetic": "strict (bitwise reference)" if args.strict
                   else "fast (pair-ring FMA lerp, within north_star tolerance)",
                   "l2": "no flush: inputs larger than L2 (2.38 GB stack + 512 MiB volume)",
                   "parallelism": f"z-slab x{world}" + (
                       "" if world == 1 else
                       " + fused slab gather (final-pass stores into rank 0's volume via CUDA IPC / NVLink)"
                       if fused else " + NCCL slab gather"),
                   "slab_bounds": [int(b) for b in bounds]},
        "gpu_launches": total_launches,
        "gpu_launches_note": "backprojection launches + pair-ring expansion launches (one per view "
                             "batch, bp_expand_kernel) inside the timed region",
        "visible_updates_per_step": visible_all,
        "gups_visible": visible_all * args.steps / (ms / 1e3) / 1e9,
        "kernel_ms_per_step": kernel_ms / args.steps,
        "value_strict_bitwise": (nominal_step * args.steps / (strict_ms / 1e3) / 1e9) if strict_ms else None,
        "value_hw_rcp": (nominal_step * args.steps / (hwr_ms / 1e3) / 1e9) if hwr_ms else None,
        "value_hw_rcp_note": "opt-in BP_RECIP_HW_APPROX (rcp.approx, no Newton step): RMS 3.3e-7 / max "
                             "2.9e-5 of max|ref| vs 7e-9 / 6.5e-6 for the headline fast mode",
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak_nominal,
                     "unit": "GB/s", "frac": achieved / peak_nominal,
                     "traffic": prof.get("dram_bytes_per_launch"),
                     "peak_source": f"nominal 128 B/clk/SM x 148 SMs at sm_max {sm_max:.0f} MHz "
                                    "(MEASURED_PEAKS.json has no shared-memory figure)",
                     "frac_at_measured_clock": achieved / (peak_nominal * float(sm_mhz) / float(sm_max)),
                     "hbm_check": {
                         "achieved": (8.0 * (z1 - z0) * L * L + tex_bytes * isx * isy * n
                                      / max(1e-9, launches_per_step)) / per_launch_s / 1e9,
                         "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                         "note": "algorithmic HBM bytes per launch (slab volume read + write, the launch's "
                                 "views: 8-byte pair-ring texels in fast mode, 4-byte raw in strict) / live "
                                 "mean launch time; ncu: profiles/latest.json. HBM is not the bound"},
                     "binding_unit": {
                         "unit": "FMA pipe at the margin (~19 lane-ops per update with exact coordinates); "
                                 "LSU shared-memory wavefronts busy but not limiting (DESIGN.md 3.5 A/Bs)",
                         "util": prof.get("fma_pipe_active_pct", 0.0) / 100.0,
                         "lsu_wavefront_util": prof.get("lsu_wavefronts_pct", 0.0) / 100.0,
                         "issue_active": prof.get("issue_active_pct", 0.0) / 100.0,
                         "source": "ncu --set full of the same kernel (profiles/latest.json)"}},
        "e2e": {"value": e2e_val, "unit": "GUP/s", "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps,
                "ms_per_step": e2e_s * 1e3 / args.steps,
                "h2d_ms_per_step": h2d_ms / args.steps, "d2h_ms_per_step": d2h_ms / args.steps,
                "ms_each": [round(x, 2) for x in e2e_each]},
        "clocks": clocks,
        "tile": {"w": st.tile_w, "h": st.tile_h, "block": [st.block_x, st.block_y, st.block_z],
                 "tile_pairs": st.tile_pairs, "skipped_pairs": st.skipped_pairs,
                 "fallback_pairs": st.fallback_pairs},
        "datagen_s": gen_s,
    }
    if e2e_pipe:
        line["e2e_pipelined"] = e2e_pipe
    if e2e_copy:
        line["e2e_copy"] = e2e_copy
    if fdk:
        line["fdk_e2e"] = fdk
    if gather_check is not None:
        line["gather_bitwise_vs_single_context"] = gather_check
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--l", "--edge", dest="l", type=int, default=512,
                    help="voxels per edge (use --edge under torchrun: its parser claims --l)")
    ap.add_argument("--views", type=int, default=496)
    ap.add_argument("--batch", type=int, default=248, help="views per launch, resident (value) run "
                    "(496 = 2 x 248)")
    ap.add_argument("--e2e-batch", type=int, default=0,
                    help="views per launch, streamed e2e run (default 32 for the whole volume, 62 for "
                         "a z-slab of a multi-GPU run: tools/scaling_projection.py)")
    ap.add_argument("--seed", type=int, default=20110428)
    ap.add_argument("--strict", action="store_true", help="bitwise reference arithmetic")
    ap.add_argument("--cpu-views", type=int, default=64,
                    help="views of the bounded CPU-baseline sample in our arm (about 10-20 s)")
    ap.add_argument("--ref-steps", type=int, default=2,
                    help="reference arm: at most this many timed full reconstructions")
    ap.add_argument("--ref-sample-views", type=int, default=0,
                    help="reference arm: time the first N views only (0: all)")
    ap.add_argument("--write-stack", default=None,
                    help="write the seeded BASELINE stack (first --sample-views views) to this "
                         "BPST path and exit")
    ap.add_argument("--sample-views", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fdk", action="store_true", help="skip the e2e run with GPU filtering")
    ap.add_argument("--no-copy-path", action="store_true",
                    help="skip the pageable copy-semantics e2e run (e2e_copy)")
    ap.add_argument("--no-pipelined", action="store_true",
                    help="skip the back-to-back (two-context) e2e run")
    ap.add_argument("--verify-gather", action="store_true",
                    help="N>1: compare rank 0's gathered volume with a single-context run")
    args = ap.parse_args()
    args.fast_off = args.strict
    if args.e2e_batch <= 0:
        args.e2e_batch = 32 if int(os.environ.get("WORLD_SIZE", "1")) == 1 else 62
    if args.write_stack:
        return write_stack(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
