#!/usr/bin/env python
"""graphvx-b200 benchmark (driver contract, see task README / DESIGN.md §6).

Default workload = BASELINE.json's headline configuration, configs[4]: the
Gaussian3x3 -> Sobel3x3 -> Magnitude graph on one 16384^2 U8 image, run as
N row bands (one per GPU / rank) through the library's BandedSession with
the halo rows exchanged over NCCL every step.  One *step* = one execution
of the graph over the whole image.  `--config k` selects the other BASELINE
configs (1..4: frame batches through DeviceSession, N ranks = N frame
replicas).

Prints ONE JSON line on rank 0.  `--impl reference` times the reference CPU
engine (oracle/_ref, built unmodified from the reference sources) on bounded
samples of the same workload instead.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG_NAME = {
    1: "Gaussian3x3->Sobel3x3->Magnitude 1920x1080 U8",
    2: "Harris corners (Sobel, Ixx/Iyy/Ixy, Box3x3, F32 response, threshold) 3840x2160 U8",
    3: "Unsharp mask with user-defined 5x5 local node 7680x4320 U8",
    4: "Gaussian5x5 (Convolve) -> ConvertDepth -> Histogram + MeanStdDev, 4K frames",
    5: "Gaussian3x3->Sobel3x3->Magnitude 16384x16384 U8, row bands + halo exchange",
}
# algorithmic HBM bytes per output pixel of the fused program
ALGO_BYTES = {1: 3, 2: 2, 3: 2, 4: 1, 5: 3}
KERNEL_NAME = {1: "edge8_kernel", 2: "harris4_kernel", 3: "sep_kernel<5,1> (separable stencil, unsharp epilogue)", 4: "sep_kernel<5,2> (separable conv + value histogram)",
               5: "edge8_kernel"}
# frames per launch: each step is one fused launch over a batch of frames; the
# two rotating batches (inputs + outputs) span >= 4x the 126 MB L2 (SURVEY.md
# §8d), which also amortises the ~20 us fixed cost of a launch (ramp + tail)
DEFAULT_FRAMES = {1: 64, 2: 32, 3: 8, 4: 64, 5: 1}
# inputs / outputs rotate over NPOOL buffer sets: a launch may overlap the
# kernels still running before it only when it touches none of their data
# (the library's overlap window, runtime.cu launch_tracked), so with NPOOL
# sets one launch in NPOOL is fully stream-ordered
NPOOL = 16
CPU_SAMPLE = {1: (1920, 1080), 2: (3840, 544), 3: (7680, 272), 4: (3840, 544), 5: (16384, 128)}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def ncu_traffic(cfg):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            data = json.load(f)
        return data.get(str(cfg))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, device: int):
        self.device, self.samples, self.proc = device, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------- CPU legs

def cpu_reference_run(cfg, steps, warmup):
    """Reference CPU engine on bounded samples of the workload (all host threads)."""
    import oracle
    kind = "reference" if oracle.have_ref() else "port"
    w, h = CPU_SAMPLE[cfg]
    img = oracle.ref_random_u8(w, h, cfg) if kind == "reference" else None
    if img is None:
        import paper_2008_11476_b200 as gvx
        img = gvx.random_u8(w, h, cfg)
    ncpu = os.cpu_count() or 1
    workers = max(1, ncpu // 4) if kind == "reference" else ncpu  # the reference engine uses <= 4 threads

    def one(_):
        if kind == "reference":
            oracle.ref_run(cfg, img)
        else:
            oracle.port_run(cfg, img)

    with ThreadPoolExecutor(workers) as ex:
        for _ in range(warmup):
            list(ex.map(one, range(workers)))
        t0 = time.perf_counter()
        for _ in range(steps):
            list(ex.map(one, range(workers)))
        dt = time.perf_counter() - t0
    px = w * h * workers * steps
    return {"value": px / dt / 1e6, "unit": "Mpixel/s", "cores": min(ncpu, 4 * workers) if kind == "reference" else ncpu,
            "kind": kind, "sample": f"{workers} concurrent x {w}x{h} crop(s) of config {cfg} per step, {steps} steps",
            "seconds": dt}


def cpu_baseline_leg(cfg):
    """~10-30 s of reference CPU work on one bounded sample (rank 0, N=1)."""
    import oracle
    kind = "reference" if oracle.have_ref() else "port"
    w, h = CPU_SAMPLE[cfg]
    if cfg in (1,):
        w, h = 1920, 1080
    import paper_2008_11476_b200 as gvx
    img = gvx.random_u8(w, h, cfg)
    reps, t_total = 0, 0.0
    while t_total < 10.0 and reps < 50:
        t0 = time.perf_counter()
        if kind == "reference":
            oracle.ref_run(cfg, img)
        else:
            oracle.port_run(cfg, img)
        t_total += time.perf_counter() - t0
        reps += 1
    return {"value": w * h * reps / t_total / 1e6, "unit": "Mpixel/s",
            "cores": min(4, os.cpu_count() or 1) if kind == "reference" else 1, "kind": kind,
            "sample": f"{reps} run_naive call(s) on a {w}x{h} crop of config {cfg} (reference uses <=4 threads)",
            "seconds": round(t_total, 3)}


# ------------------------------------------------------------------ GPU legs

def make_frames(gvx, w, h, n, seed):
    base = gvx.random_u8(w, h, seed)
    frames = [base]
    for i in range(1, n):
        frames.append(np.roll(base, shift=(i * 7919) % (w * h)).reshape(h, w) ^ np.uint8((i * 37) & 0xFF))
    return np.stack(frames)


def run_frames(args, cfg, rank, world, local_rank):
    import paper_2008_11476_b200 as gvx
    w, h = gvx.CONFIG_SIZE[cfg]
    F = args.frames or DEFAULT_FRAMES[cfg]
    dev = gvx.Device(local_rank)
    graph = gvx.ConfigGraph(cfg, w, h, True)
    sess = gvx.Session(graph, frames=F)
    sess.set_stream(dev.stream)
    sess.set_overlap(1)  # only this session launches kernels on dev.stream
    pitch = (w + 127) // 128 * 128
    in_bytes = pitch * h * F
    out_pitch = pitch * (2 if cfg in (1, 5) else 1)
    pools = []
    host = make_frames(gvx, w, h, F, gvx.CONFIG_SEED[cfg] + 97 * rank)
    # end to end through the public API (host buffers in and out, H2D + D2H
    # inside), measured first, on a quiet device
    # --e2e-frames 0 (profiling runs only) skips this leg
    e2e_frames = args.e2e_frames
    e2e = None
    if e2e_frames > 0:
        # frames stream through gvx::HostPipeline: frame k+1's upload, frame k's
        # kernels and frame k-1's download overlap; every result is read back
        depth = int(os.environ.get("GVX_E2E_DEPTH", 3))  # frames in flight; measured best of 2 / 3 / 4 / 6
        pipe = gvx.Pipeline(graph, depth=depth)
        out_host = graph.output_array()
        # the input frames live in page-locked host memory (registered once,
        # outside the timed region): every frame is still DMAed host->device
        # inside it, without a staging copy
        pinned = gvx.PinnedHost([host])
        for i in range(max(depth + 1, F)):  # warm: staging, contexts, modules, every registered frame's first DMA
            if pipe.pending() >= depth:
                pipe.next(out_host)
            pipe.submit(host[i % F], pinned=True)
        while pipe.pending():
            pipe.next(out_host)
        view = cfg != 4  # image results are read in place from page-locked staging
        stream = [host[i % F] for i in range(e2e_frames)]
        for rep in range(2):  # rep 0: untimed warm-up pass of the same loop
            barrier()
            t0 = time.perf_counter()
            if view:  # one native call: submit / take loop in C++ (gvxc_pipeline_stream)
                pipe.stream(stream, pinned=True)
            else:
                for i in range(e2e_frames):
                    if pipe.pending() >= depth:
                        pipe.next(out_host)
                    pipe.submit(host[i % F], pinned=True)
                while pipe.pending():
                    pipe.next(out_host)
        e2e_s = allreduce_max(time.perf_counter() - t0)
        e2e_value = w * h * e2e_frames * world / e2e_s / 1e6
        out_b = {1: 2, 2: 1, 3: 1, 4: 256 * 8 + 16, 5: 2}[cfg]
        e2e = {"value": e2e_value, "unit": "Mpixel/s", "h2d_bytes_per_step": w * h,
               "d2h_bytes_per_step": out_b * (w * h if cfg != 4 else 1), "frames": e2e_frames,
               "path": "gvx::HostPipeline (run_plan semantics, 3 frames in flight) via gvx_c.h "
                       "(gvxc_pipeline_stream: one call for the stream): page-locked host frame in (DMA, no "
                       "staging copy), every result DMAed to page-locked host memory, in submission order"}
        del pipe
        pinned.close()

    for b in range(NPOOL):
        din = dev.alloc(in_bytes)
        for f in range(F):
            dev.upload(din + f * pitch * h, pitch, np.roll(host[f], b * 13, axis=1))
        dout = dev.alloc(out_pitch * h * F) if cfg != 4 else None
        pools.append((din, dout))
    # cfg4 outputs (histogram / mean / stddev) stay session-owned value slots

    def bind(b):
        din, dout = pools[b]
        sess.bind(0, din, pitch, pitch * h)
        if dout is not None:
            sess.bind(1, dout, out_pitch, out_pitch * h)

    for i in range(args.warmup):
        bind(i % NPOOL)
        sess.launch()
    sess.sync()
    # correctness spot check of frame 0 of the first batch against the oracle port
    checked = None
    if rank == 0 and not args.no_check:
        bind(0)
        sess.launch()
        sess.sync()
        checked = check_frame0(cfg, host[0], sess.download(0))

    ev = [dev.event() for _ in range(2)]
    barrier()
    dev.sync()
    with ClockSampler(local_rank) as clk:
        # identical load for ~1 s so nvidia-smi samples clocks under load
        # (the sampler runs across this window and the timed region)
        t_end = time.perf_counter() + args.clock_window
        i = 0
        while time.perf_counter() < t_end:
            bind(i % NPOOL)
            sess.launch()
            i += 1
            if i % 50 == 0:
                dev.sync()
        dev.sync()
        launches0 = gvx.launch_count()
        dev.record(ev[0])
        for i in range(args.steps):
            bind(i % NPOOL)
            sess.launch()
        dev.record(ev[1])
        dev.sync()
    ms = dev.elapsed_ms(ev[0], ev[1])
    launches = gvx.launch_count() - launches0
    ms_max = allreduce_max(ms)
    px_step = w * h * F
    value = px_step * args.steps * world / (ms_max / 1e3) / 1e6

    # one frame per launch (vxProcessGraph semantics: one graph execution per
    # call), device time per execution over distinct frames (> 4x L2 in turn)
    single = None
    if not args.no_single:
        s1 = gvx.Session(graph, frames=1)
        s1.set_stream(dev.stream)
        s1.set_overlap(1)
        fstride = pitch * h
        ofs = out_pitch * h

        def bind1(i):
            b, f = (i // F) % NPOOL, i % F
            din, dout = pools[b]
            s1.bind(0, din + f * fstride, pitch, fstride)
            if dout is not None:
                s1.bind(1, dout + f * ofs, out_pitch, ofs)

        n1 = max(2 * F, 64)
        for i in range(8):
            bind1(i)
            s1.launch()
        dev.sync()
        dev.record(ev[0])
        for i in range(n1):
            bind1(i)
            s1.launch()
        dev.record(ev[1])
        dev.sync()
        ms1 = dev.elapsed_ms(ev[0], ev[1]) / n1
        single = {"ms_per_frame": round(ms1, 5), "value": round(w * h / (ms1 / 1e3) / 1e6, 1), "unit": "Mpixel/s",
                  "launches_per_frame": s1.launches(), "frames_timed": n1,
                  "note": "one graph execution (one fused launch) per frame, as vxProcessGraph / run_plan "
                          "execute; inputs rotate over the same batches"}
        s1.close()

    # the drop-in host entry point itself: run_plan(plan, InputMap) on pageable
    # host buffers, one call per frame (copies in and out inside each call)
    run_plan_e2e = None
    if not args.no_single:
        g2 = gvx.ConfigGraph(cfg, w, h, True)
        dst = g2.output_array()  # the caller's destination, reused across frames
        for i in range(2):  # the second call page-locks the recycled output vectors
            g2.run_host(host[i % F], out=dst)
        n2 = 8
        t0 = time.perf_counter()
        for i in range(n2):
            g2.run_host(host[i % F], out=dst)
        dt = time.perf_counter() - t0
        run_plan_e2e = {"value": round(w * h * n2 / dt / 1e6, 1), "unit": "Mpixel/s", "frames": n2,
                        "path": "gvx::run_plan(plan, InputMap) via gvxc_graph_run_host: pageable numpy frame in, "
                                "output copied to the caller's numpy array, one synchronous call per frame"}
        g2.close()

    # one fused launch per step (F frames in grid.z); a cfg4 batch also holds
    # the scratch-clear and MeanStdDev-finalize micro-kernels (counted in, so
    # the roofline fraction is a lower bound for the conv/histogram kernel;
    # a single frame is one launch: its last CTA finalizes)
    kernel_ms = ms / args.steps
    if sess.launches() != 1 and cfg != 4:
        kernel_ms = None
    return dict(value=value, ms_per_step=ms_max / args.steps, clocks=clk.summary(), launches=launches,
                e2e=e2e, frames=F, kernel_ms=kernel_ms, checked=checked, w=w, h=h, px_step=px_step,
                launches_per_step=sess.launches(), describe=graph.describe(), single_frame=single,
                run_plan_e2e=run_plan_e2e)


# --------------------------------------------------------------- banded cfg5

def check_frame0(cfg, frame, got):
    """Frame 0 (the reference's random_buffer input of the config's seed)
    against the unmodified reference's run_naive output at the configured
    size: SHA-256 digests / exact statistics in tests/golden/fullsize.json.
    None when the frame is not that input."""
    import hashlib
    fx = fullsize_fixture(cfg)
    if not fx or frame.shape != (fx["height"], fx["width"]):
        return None
    sha = hashlib.sha256(np.ascontiguousarray(frame).tobytes()).hexdigest()
    if cfg == 4:
        f0 = fx["frames"][0]
        if sha != f0["input_sha256"]:
            return None
        hist, mean, sd = got
        return bool(list(hist) == f0["hist"] and mean == float.fromhex(f0["mean"]) and sd == float.fromhex(f0["stddev"]))
    if sha != fx["input_sha256"]:
        return None
    return hashlib.sha256(np.ascontiguousarray(got).tobytes()).hexdigest() == fx["output_sha256"]


def fullsize_fixture(cfg):
    try:
        with open(os.path.join(REPO, "tests", "golden", "fullsize.json")) as f:
            return json.load(f).get(str(cfg))
    except Exception:
        return None


def run_banded(args, rank, world, local_rank):
    """cfg5: the 16384^2 edge graph as `world` row bands through the library
    (gvx::BandedSession via gvx_c.h).  Each rank holds its owned input rows;
    every step the band's 2 halo rows per neighbour arrive over NCCL
    (gvxb_halo_start, issued by the library) while the interior rows run,
    then the edge rows.  No torch on this path."""
    import hashlib
    import paper_2008_11476_b200 as gvx
    W = H = args.size or 16384
    comm = gvx.Comm(rank, world, local_rank) if world > 1 else None
    global _comm
    _comm = comm
    dev = gvx.Device(local_rank)
    graph = gvx.ConfigGraph(5, W, H, True)
    band = gvx.Band(graph, rank, world, comm, device=local_rank)
    band.set_stream(dev.stream)
    L = band.layout
    r0, r1, s0, s1 = L["row0"], L["row1"], L["src_row0"], L["src_row1"]
    # the reference's random_buffer input (seed 5); this rank
    # uploads only the rows it owns: its halo rows come from the exchange
    img = gvx.random_u8(W, H, 5)
    band.upload(0, img[r0:r1], r0)
    # results rotate over NPOOL output buffers (as the frame configs rotate
    # their batches): an execution overlaps the ones still running before it
    # when it touches none of their data (programmatic dependent launch; only
    # this band's work runs on dev.stream)
    band.set_overlap(1)
    out_pitch = (2 * W + 127) // 128 * 128
    outs = [dev.alloc(out_pitch * (r1 - r0)) for _ in range(NPOOL)]

    def launch(i):
        band.bind(1, outs[i % NPOOL], out_pitch, out_pitch * (r1 - r0))
        band.launch()

    for i in range(args.warmup):
        launch(i)
    band.sync()
    launch(0)
    band.sync()
    checked = None
    if not args.no_check:
        # bit-exact vs the reference: SHA-256 digests of oracle/_ref run_naive
        # over the same input (tests/golden/fullsize.json), per 2048-row block;
        # every rank joins the all-reduce (2 = its band is not block-aligned)
        fx = fullsize_fixture(5)
        verdict = 2.0
        if fx and fx["width"] == W and fx["height"] == H and r0 % fx["block_rows"] == 0 and \
                (r1 % fx["block_rows"] == 0 or r1 == H):
            out = band.download(1, r0, r1 - r0, np.int16)
            br = fx["block_rows"]
            ok = all(hashlib.sha256(out[a - r0:a - r0 + br].tobytes()).hexdigest() == fx["block_sha256"][a // br]
                     for a in range(r0, r1, br))
            verdict = 0.0 if ok else 1.0
            del out
        worst = allreduce_max(verdict)
        checked = None if worst == 2.0 else worst == 0.0
    ev = [dev.event() for _ in range(2)]
    barrier()
    dev.sync()
    with ClockSampler(local_rank) as clk:
        t_end = time.perf_counter() + args.clock_window
        i = 0
        while time.perf_counter() < t_end:
            launch(i)
            i += 1
            if i % 20 == 0:
                dev.sync()
        dev.sync()
        barrier()
        launches0 = gvx.launch_count()  # every context of the process (the band has its own)
        dev.record(ev[0])
        for i in range(args.steps):
            launch(i)
        dev.record(ev[1])
        dev.sync()
    ms = dev.elapsed_ms(ev[0], ev[1])
    ms_max = allreduce_max(ms)
    value = W * H * args.steps / (ms_max / 1e3) / 1e6
    launches = gvx.launch_count() - launches0
    # e2e through the same API: BandedSession::run_host streams the rank's
    # input slab (owned + halo rows, page-locked) up and its magnitude rows
    # down in 1024-row pieces (upload, kernel, download overlapped on three
    # streams); the halo rows come with the host slab, so no exchange
    src = gvx.HostBuffer((s1 - s0, W), np.uint8)
    src.array[:] = img[s0:s1]
    dst = gvx.HostBuffer((r1 - r0, W), np.int16)
    # the drop-in host entry point at N=1: run_plan(plan, InputMap) with the
    # whole 16384^2 frame in pageable host memory, one synchronous call
    run_plan_e2e = None
    if world == 1 and not args.no_single:
        dst_frame = graph.output_array()  # the caller's destination, reused across frames
        for _ in range(2):  # the second call page-locks the recycled output vectors
            graph.run_host(img, out=dst_frame)
        n2 = 3
        t0 = time.perf_counter()
        for _ in range(n2):
            graph.run_host(img, out=dst_frame)
        dt = time.perf_counter() - t0
        run_plan_e2e = {"value": round(W * H * n2 / dt / 1e6, 1), "unit": "Mpixel/s", "frames": n2,
                        "path": "gvx::run_plan(plan, InputMap) via gvxc_graph_run_host: pageable 268 MB frame in, "
                                "537 MB magnitude copied out to the caller's array, one synchronous call per frame"}
        del dst_frame
    del img
    band.run_host(src.ptr, W, 1, dst.ptr, 2 * W, 1024)  # warm-up
    n_e2e = max(3, min(args.steps, 5))
    barrier()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        band.run_host(src.ptr, W, 1, dst.ptr, 2 * W, 1024)
    e2e_s = allreduce_max(time.perf_counter() - t0)
    e2e_ok = None
    if not args.no_check:
        want = band.download(1, r0, r1 - r0, np.int16)
        e2e_ok = bool(np.array_equal(want, dst.array))
    e2e = {"value": W * H * n_e2e / e2e_s / 1e6, "unit": "Mpixel/s", "h2d_bytes_per_step": (s1 - s0) * W,
           "d2h_bytes_per_step": (r1 - r0) * W * 2, "checked_vs_device_result": e2e_ok,
           "path": "gvx::BandedSession::run_host via gvx_c.h (gvxc_band_run_host): page-locked input slab rows in, "
                   "magnitude rows out, 1024-row pieces with upload / kernel / download overlapped on three streams"}
    src.close()
    dst.close()
    return dict(value=value, ms_per_step=ms_max / args.steps, clocks=clk.summary(), launches=launches, e2e=e2e,
                frames=1, kernel_ms=ms / args.steps if world == 1 else None, checked=checked, w=W, h=H,
                px_step=W * H, launches_per_step=band.launches(), describe=band.describe(),
                run_plan_e2e=run_plan_e2e)


# ------------------------------------------------------------- distributed

_dist = None
_comm = None  # gvx.Comm (library NCCL communicator) on the banded path


def init_dist(world, local_rank, cfg):
    """Frame replicas (cfg1-4) use torch.distributed for the barrier and the
    max-over-ranks timing; the banded cfg5 path uses the library's own NCCL
    communicator (created in run_banded) and never imports torch."""
    global _dist
    if world <= 1 or cfg == 5:
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    _dist = dist


def barrier():
    if _comm is not None:
        _comm.barrier()
    elif _dist is not None:
        _dist.barrier()


def allreduce_max(x: float) -> float:
    if _comm is not None:
        return _comm.allreduce_max(x)
    if _dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    _dist.all_reduce(t, op=_dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="graphvx-b200", choices=["graphvx-b200", "ours", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--size", type=int, default=0, help="cfg5 image side (default 16384)")
    ap.add_argument("--e2e-frames", type=int, default=48)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single", action="store_true", help="skip the one-frame-per-launch and run_plan legs")
    ap.add_argument("--clock-window", type=float, default=1.0, help="seconds of identical load sampled before timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local_rank = dist_env()
    cfg = args.config
    import paper_2008_11476_b200 as gvx
    w, h = gvx.CONFIG_SIZE[cfg]

    if args.impl == "reference":
        if rank != 0:
            return 0
        r = cpu_reference_run(cfg, args.steps, args.warmup)
        line = {"metric": "graph Mpixel/s", "value": r["value"], "unit": "Mpixel/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": r["seconds"] / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong" if cfg == 5 else "weak",
                "vs_baseline": None, "dtype": "u8", "data": "synthetic (reference random_buffer)",
                "config": {"workload": CONFIG_NAME[cfg], "width": w, "height": h},
                "impl": "reference", "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "gpu_launches": 0}
        print(json.dumps(line), flush=True)
        return 0

    os.environ.setdefault("GVX_DEVICE", str(local_rank))
    init_dist(world, local_rank, cfg)
    if cfg == 5:
        res = run_banded(args, rank, world, local_rank)
        scaling = "strong"
    else:
        res = run_frames(args, cfg, rank, world, local_rank)
        scaling = "weak"
    if rank != 0:
        return 0

    peaks, peak_kind = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    roof = None
    if res["kernel_ms"]:
        achieved = ALGO_BYTES[cfg] * res["px_step"] / (res["kernel_ms"] / 1e3) / 1e9
        prof = ncu_traffic(cfg) or {}
        traffic = None
        if prof.get("dram_bytes_per_launch") and prof.get("px_per_launch"):
            # per launch of this run (the capture used the same command; scale if frames differ)
            traffic = round(prof["dram_bytes_per_launch"] * res["px_step"] / prof["px_per_launch"])
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_kind,
                "kernel": KERNEL_NAME[cfg], "algorithmic_bytes_per_px": ALGO_BYTES[cfg],
                "px_per_launch": res["px_step"], "kernel_ms": round(res["kernel_ms"], 4)}
        if prof.get("warp_inst_per_px"):
            # the kernels are issue-bound: lane instructions/s against 148 SMs x 4 schedulers x 32 lanes x clock
            mhz = (res.get("clocks") or {}).get("sm_mhz") or 1965.0
            lane_rate = prof["warp_inst_per_px"] * 32 * res["px_step"] / (res["kernel_ms"] / 1e3)
            issue_peak = 148 * 4 * 32 * mhz * 1e6
            roof["issue"] = {"warp_inst_per_px": prof["warp_inst_per_px"], "lane_inst_per_s": round(lane_rate),
                             "peak": round(issue_peak), "frac": round(lane_rate / issue_peak, 4),
                             "source": prof.get("source")}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_leg(cfg)
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)}
    line = {"metric": "graph Mpixel/s", "value": res["value"], "unit": "Mpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (reference random_buffer, seed 5)" if cfg == 5 else
                    "synthetic (reference random_buffer frame + derived frames)",
            "config": {"workload": CONFIG_NAME[cfg], "width": res["w"], "height": res["h"],
                       "frames_per_step": res["frames"], "l2": f"inputs/outputs rotate over {NPOOL} batches spanning >= 4x L2"
                       if cfg != 5 else "16384^2 input > L2",
                       "parallelism": f"{'row bands' if cfg == 5 else 'frame replicas'} x{world}"},
            "e2e": res["e2e"], "roofline": roof, "cpu_baseline": cpu, "clocks": res["clocks"],
            "gpu_launches": res["launches"], "launches_per_step": res["launches_per_step"],
            "single_frame": res.get("single_frame"), "run_plan_e2e": res.get("run_plan_e2e"),
            "checked_vs_oracle": res["checked"],
            "checked_against": "SHA-256 of oracle/_ref run_naive (unmodified reference) per 2048-row block"
                               if cfg == 5 else "oracle/_ref run_naive (unmodified reference) on frame 0: SHA-256 of "
                               "the output (histogram / mean / stddev for cfg4), tests/golden/fullsize.json",
            "program": res["describe"]}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
