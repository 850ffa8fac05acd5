#!/usr/bin/env python
"""Benchmark: cardiac-cine SENSE reconstruction (BASELINE.json configs[2], C3).

One step = reconstruct one 256x256 x 32-coil x 30-frame cine end to end:
k-space from pinned host memory -> H2D -> fused IFFT2 + conj-sensitivity coil
combine -> D2H -> images in pinned host memory, through the public streaming
API (hetreco_stream_run).  Under torchrun the 30 frames are split into
contiguous frame slabs over the ranks (strong scaling, no collective on the
data path); rank r streams only its slab.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  `value` = `e2e.value` = frames/s of the whole
volume (device time between CUDA events on each rank's compute stream, which
the pipeline joins after its last D2H; max over ranks).  Side fields:
`device_resident` (the same chain with the slab already in HBM), `roofline`
(the dominant kernel against MEASURED_PEAKS.json), `weak_scaling` (N > 1:
every rank a whole volume), `cpu_baseline` (the reference library,
oracle/_ref, through its own ComputeSession API on this host's cores) and
`other_configs` (C1, C2, C4 resident; C5 streamed and sharded like C3).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NX, NY, NC, NF = 256, 256, 32, 30
METRIC = "recon frames/s end-to-end incl. H2D/D2H at 1/2/4/8 GPU; kernel HBM GB/s vs peak"
UNIT = "frames/s"
CONFIG = {"workload": "C3 cardiac cine SENSE: 256x256 k-space, 32 coils x 30 frames (one volume; "
                      "frames sharded over the GPUs), IFFT2 + conj-sensitivity coil combine",
          "nx": NX, "ny": NY, "coils": NC, "frames": NF, "dtype_io": "complex64",
          "l2_policy": "inputs (496 MiB/step) larger than L2 (126 MB); no flush"}
# algorithmic bytes (SURVEY.md §8 d): Y 16 MiB + M 0.5 MiB per frame, S 16 MiB once per launch
FRAME_Y = NX * NY * NC * 8
FRAME_M = NX * NY * 8
SMAP = NX * NY * NC * 8
C5_NX, C5_NC = 512, 32


def config_for(world: int) -> dict:
    """The config dict both arms print (identical keys and values)."""
    return dict(CONFIG, parallelism=f"frame-slab x{world} (no collective)")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the timed regions run."""

    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap", "gpu_idle"]
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,clocks_event_reasons.gpu_idle")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._on = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        while not self._stop.is_set():
            if self._on.wait(0.05) and not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out and self._on.is_set():
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.05)

    def on(self):
        self._on.set()

    def off(self):
        self._on.clear()

    def close(self):
        self._stop.set()
        self._on.set()
        self._t.join()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({n for r in self.rows for i, n in enumerate(self.REASONS)
                          if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HETRECO_BENCH_DEVICE pins every rank to one GPU (with
    # HETRECO_BENCH_DIST=gloo): a dry run of the multi-rank path on a 1-GPU box
    if os.environ.get("HETRECO_BENCH_DEVICE"):
        local = int(os.environ["HETRECO_BENCH_DEVICE"])
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("HETRECO_BENCH_DIST", "nccl")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def reduce_max(x: float, world: int) -> float:
    from paper_1807_11830_b200.sharding import max_over_ranks
    return max_over_ranks(x) if world > 1 else x


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def fill_frames(Y, first: int):
    """Y[..., i] = C3 frame first + i (seeded per frame, so every rank makes
    exactly its own slab of the same volume)."""
    for i in range(Y.shape[3]):
        rng = np.random.default_rng([1234, first + i])
        Y[..., i] = (rng.standard_normal((NX, NY, NC), dtype=np.float32)
                     + 1j * rng.standard_normal((NX, NY, NC), dtype=np.float32))
    return Y


def make_maps():
    rng = np.random.default_rng(99)
    G = (rng.standard_normal((NX, NY, NC), dtype=np.float32) + 1j * rng.standard_normal((NX, NY, NC), dtype=np.float32))
    return np.asfortranarray((G / np.sqrt((np.abs(G) ** 2).sum(axis=2, keepdims=True))).astype(np.complex64))


def make_inputs():
    """The whole C3 volume in pageable memory (reference arm / CPU baseline)."""
    Y = fill_frames(np.empty((NX, NY, NC, NF), np.complex64, order="F"), 0)
    return Y, make_maps()


def cpu_baseline(Y, S, budget_s: float = 10.0):
    """The reference library itself (oracle/_ref) on all 30 C3 frames per launch."""
    from oracle import oracle as o
    if o.reference_available():
        kind = "reference"
        _, t1, _ = o.ref_recon("sens", Y, S, reps=1)  # warm-up + estimate
        reps = max(2, min(50, int(budget_s / max(t1, 1e-3))))
        _, mean_s, _ = o.ref_recon("sens", Y, S, reps=reps)
        cores = o.ref_pool_threads()
    else:  # reference not built on this host: single-thread C port
        kind = "port"
        t0 = time.perf_counter()
        o.sens_recon(Y, S)
        mean_s = time.perf_counter() - t0
        reps, cores = 1, 1
    return {"value": NF / mean_s, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"all 30 C3 frames (256x256x32 coils) per launch, {reps} launches, plan baked once; "
                      f"WorkerPool threads = min(hw, 16), host has {os.cpu_count()} cores",
            "seconds_per_frame": mean_s / NF}


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference library driven through its ComputeSession API) on the same
    workload as our arm.  One step = register the k-space of all 30 frames (the
    reference's H2D), run the SENSE chain (fft_radix2_pass x18 +
    complex_element_prod + ximage_sum), fetch the images (D2H); sensitivity
    maps and the FFT plan are set up once, as on the B200 arm.  Under torchrun
    rank 0 alone runs it (one CPU implementation per host)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as o
    Y, S = make_inputs()
    if o.reference_available():
        kind = "reference"
        o.ref_recon_e2e("sens", Y, S, reps=max(1, min(args.warmup, 2)))
        _, mean_s = o.ref_recon_e2e("sens", Y, S, reps=args.steps)
        cores = o.ref_pool_threads()
    else:
        kind = "port"
        o.sens_recon(Y, S)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            o.sens_recon(Y, S)
        mean_s = (time.perf_counter() - t0) / args.steps
        cores = 1
    value = NF / mean_s
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (complex64 I/O, fp32 FFT, fp64 coil accumulation)",
            "data": "synthetic (seeded N(0,1) k-space, normalised random sensitivity maps)",
            "config": config_for(int(os.environ.get("WORLD_SIZE", "1"))), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": "all 30 C3 frames per step: register_data(k-space) + fft_radix2_pass x18 + "
                                       "complex_element_prod + ximage_sum + fetch_data; "
                                       f"WorkerPool threads = min(hw,16) of {os.cpu_count()} host cores"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    from paper_1807_11830_b200 import hetreco as h
    from paper_1807_11830_b200.sharding import frame_slab, imbalance

    rank, world, local = dist_setup()
    # host placement: this rank's thread and pinned buffers on its GPU's NUMA node
    # (the CPU-baseline leg below gets the whole host back)
    all_cpus = os.sched_getaffinity(0)
    numa_node = h.bind_to_device_numa(local)
    devs = h.enumerate_devices()  # descriptors only: no context on the other GPUs
    s = h.ComputeSession(device=next(d for d in devs if d.backend_id == f"cuda{local}"))
    # strong scaling: one 30-frame volume, rank r owns frames [b, e)
    fb, fe = frame_slab(rank, world, NF)
    nfr = fe - fb
    S = make_maps()
    Yp = fill_frames(h.pinned_empty((NX, NY, NC, nfr), np.complex64), fb)
    Mp = h.pinned_empty((NX, NY, nfr), np.complex64)
    chunk = max(1, min(args.chunk, (nfr + 1) // 2))
    st = h.StreamingRecon(s, "sense", NX, NY, NC, chunk, S)
    chunks_per_run = (nfr + chunk - 1) // chunk
    sampler = ClockSampler(local)

    # ---- headline: end to end through the public streaming API -----------------------
    # pinned k-space slab -> H2D (copy stream) -> fused IFFT2 + SENSE -> D2H
    # (second copy stream) -> pinned image slab, every step inside the timed
    # region; device time between CUDA events on the session's compute stream
    # (the pipeline joins it after the last D2H), max over ranks.
    sampler.on()
    t_end = time.perf_counter() + 0.5
    n = 0
    while n < args.warmup or time.perf_counter() < t_end:
        st.run(Yp, Mp)
        n += 1
    barrier(world)
    w0 = time.perf_counter()
    s.timer_start()
    for _ in range(args.steps):
        st.run(Yp, Mp)
    t_e2e = s.timer_stop()
    wall_e2e = time.perf_counter() - w0
    barrier(world)
    sampler.off()
    t_e2e_max = reduce_max(t_e2e, world)
    wall_e2e_max = reduce_max(wall_e2e, world)
    value = NF * args.steps / t_e2e_max
    e2e = {"value": value, "unit": UNIT, "h2d_bytes_per_step": FRAME_Y * NF, "d2h_bytes_per_step": FRAME_M * NF,
           "h2d_bytes_per_step_per_rank": FRAME_Y * nfr, "chunk_frames": chunk,
           "wall_value": NF * args.steps / wall_e2e_max,
           "host_link_gbs_per_rank": FRAME_Y * nfr * args.steps / t_e2e / 1e9,
           "note": "hetreco_stream_run over this rank's pinned frame slab; sensitivity maps uploaded once at "
                   "init (resident), k-space H2D and images D2H per step"}

    # ---- device-resident side measurement (same slab, data already in HBM) -----------
    hin = s.register_data(h.Data([np.asfortranarray(Yp), S], h.DataKind.KData))
    hout = s.allocate_data([((NX, NY, nfr), np.complex64)], h.DataKind.XData)
    p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init()
    sampler.on()
    t_end = time.perf_counter() + 0.5
    n = 0
    while n < args.warmup or time.perf_counter() < t_end:
        p.launch()
        n += 1
        if n % 50 == 0:
            s.synchronize()
    s.synchronize()
    barrier(world)
    s.timer_start()
    dev_steps = max(args.steps, 50)
    for _ in range(dev_steps):
        p.launch()
    t_dev = s.timer_stop()
    barrier(world)
    sampler.off()
    t_dev_max = reduce_max(t_dev, world)
    M_dev = s.fetch_data(hout).arrays[0]
    e2e["matches_resident"] = bool(np.abs(M_dev - Mp).max() <= 1e-5 * np.abs(M_dev).max())
    device_resident = {"value": NF * dev_steps / t_dev_max, "unit": UNIT, "steps": dev_steps,
                       "ms_per_step": t_dev_max / dev_steps * 1e3,
                       "note": "sens_recon process over the rank's slab resident in HBM (no host transfers)"}
    # the reference's rounding (fp32 products, fp64 coil-ordered sums, ximage_sum.cl.src:6-23) timed too
    p64 = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init({"accumulate": "fp64"})
    for _ in range(max(args.warmup, 3)):
        p64.launch()
    s.synchronize()
    barrier(world)
    s.timer_start()
    for _ in range(20):
        p64.launch()
    t64 = reduce_max(s.timer_stop(), world)
    barrier(world)
    device_resident["fp64_accumulate"] = {"value": NF * 20 / t64, "unit": UNIT, "ms_per_step": t64 / 20 * 1e3,
                                          "note": "same chain with accumulate=fp64 (the reference combine's "
                                                  "rounding; bit-exact combine given the same X)"}
    del p64

    # per-kernel device times (events between kernels on the compute stream)
    prof = p.profile(reps=10)  # [axis1, combine] per frame chunk (one chunk by default)
    k_axis1, k_axis0 = sum(prof[0::2]), sum(prof[1::2])
    bytes_axis1 = 2 * FRAME_Y * nfr                 # read Y, write X
    bytes_axis0 = FRAME_Y * nfr + SMAP + FRAME_M * nfr  # read X + S, write M
    peak, peak_kind = peaks()
    kernels = [
        {"name": "k_fft_strided_ring<256,+1,16,2,32> (axis-1 IFFT, 32-column tiles through a 2-stage cp.async "
                 "shared-memory ring)", "seconds": k_axis1, "bytes": bytes_axis1, "gbs": bytes_axis1 / k_axis1 / 1e9},
        {"name": "k_fft_combine_ss<256,4> (axis-0 IFFT + conj(S) coil combine, map rows staged in smem)",
         "seconds": k_axis0, "bytes": bytes_axis0, "gbs": bytes_axis0 / k_axis0 / 1e9},
    ]
    for k in kernels:
        k["frac"] = k["gbs"] / peak
        k["share"] = k["seconds"] / (k_axis1 + k_axis0)
    dom = max(kernels, key=lambda k: k["seconds"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and nfr == NF:
        tj = json.load(open(tp))
        traffic = tj.get("per_launch_bytes", {}).get("axis1" if dom is kernels[0] else "axis0")
    algo_step = nfr * (FRAME_Y + FRAME_M) + SMAP
    roofline = {"bound": "hbm", "achieved": dom["gbs"], "peak": peak, "unit": "GB/s", "frac": dom["frac"],
                "traffic": traffic, "peak_source": peak_kind, "kernel": dom["name"],
                "kernels": kernels, "frames_per_launch": nfr,
                "chain_achieved": algo_step / (t_dev / dev_steps) / 1e9,
                "chain_frac": algo_step / (t_dev / dev_steps) / 1e9 / peak,
                "algorithmic_bytes_per_step": algo_step}

    # host-link roofline: plain pinned H2D copy of the same bytes on this GPU
    link = h.CudaBackend(local)
    buf = link.allocate(Yp.nbytes)
    flat = Yp.reshape(-1, order="F").view(np.uint8)
    link.upload(buf, 0, flat)
    t0 = time.perf_counter()
    for _ in range(3):
        link.upload(buf, 0, flat)
    link_gbs = 3 * Yp.nbytes / (time.perf_counter() - t0) / 1e9
    link.release(buf)
    link.close()
    e2e["host_link_peak_gbs_per_rank"] = link_gbs
    e2e["host_link_frac"] = e2e["host_link_gbs_per_rank"] / link_gbs
    e2e["host_link_roofline_frames_per_s"] = world * link_gbs * 1e9 / FRAME_Y
    s.release_data(hin)
    s.release_data(hout)

    # weak scaling side field: every rank streams a whole 30-frame volume
    weak = None
    if world > 1 and not args.no_weak:
        Yw = fill_frames(h.pinned_empty((NX, NY, NC, NF), np.complex64), 0)
        Mw = h.pinned_empty((NX, NY, NF), np.complex64)
        stw = h.StreamingRecon(s, "sense", NX, NY, NC, args.chunk, S)
        stw.run(Yw, Mw)
        barrier(world)
        s.timer_start()
        wsteps = max(3, min(args.steps, 20))
        for _ in range(wsteps):
            stw.run(Yw, Mw)
        tw = reduce_max(s.timer_stop(), world)
        weak = {"value": world * NF * wsteps / tw, "unit": UNIT, "frames_per_gpu": NF, "steps": wsteps}
        del stw, Yw, Mw

    # the reference-shaped flow (rank 0, N=1): register pageable k-space + maps,
    # launch, fetch, release per step
    if rank == 0 and world == 1 and not args.no_session_flow:
        Y = np.asfortranarray(Yp)
        hout = s.allocate_data([((NX, NY, NF), np.complex64)], h.DataKind.XData)
        hs = s.register_data(h.Data([Y], h.DataKind.KData))
        s.release_data(hs)
        Mh = np.empty((NX, NY, NF), np.complex64, order="F")
        ps = None
        t0 = time.perf_counter()
        for _ in range(5):
            hk = s.register_data(h.Data([Y, S], h.DataKind.KData))
            if ps is None:
                ps = h.Process(s, "sens_recon").set_input(hk).set_output(hout).init()
            else:
                ps.set_input(hk)
            ps.launch()
            s.fetch_data(hout, [Mh])
            s.release_data(hk)
        t_sess = (time.perf_counter() - t0) / 5
        s.release_data(hout)
        e2e["session_api_pageable"] = {
            "value": NF / t_sess, "unit": UNIT, "ms_per_step": t_sess * 1e3,
            "h2d_bytes_per_step": FRAME_Y * NF + SMAP, "d2h_bytes_per_step": FRAME_M * NF,
            "note": "register_data(pageable k-space + maps) + sens_recon launch + fetch_data per step "
                    "(the --impl reference flow); pinned staging ring on the host side"}

    # C5 (all ranks): 512^2 x 32 coils, args.c5_frames frames sharded over the
    # ranks, streamed from pinned memory
    c5 = None
    if args.c5_frames > 0 and not args.no_extras:
        c5 = c5_stream(h, s, rank, world, args.c5_frames, sampler)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.sched_setaffinity(0, all_cpus)
        Yc, Sc = make_inputs()
        cpu = cpu_baseline(Yc, Sc)
        del Yc

    extras = None
    if rank == 0 and not args.no_extras:
        extras = other_configs(h, s, peak)
        if c5:
            extras["C5_stream_rss_512x512x32"] = c5
    sampler.close()
    clocks = sampler.summary()

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_e2e_max / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 (complex64 I/O, fp32 FFT and coil accumulation)",
                "data": "synthetic (seeded N(0,1) k-space, normalised random sensitivity maps)",
                "config": config_for(world),
                "sharding": {"frames_per_gpu": [frame_slab(r, world, NF)[1] - frame_slab(r, world, NF)[0]
                                                for r in range(world)],
                             "slab_imbalance": imbalance(world, NF), "host_numa_node_rank0": numa_node},
                "impl": "hetreco-b200",
                "e2e": e2e, "device_resident": device_resident, "weak_scaling": weak,
                "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
                "gpu_launches": 2 * chunks_per_run * args.steps, "other_configs": extras}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def c5_stream(h, s, rank: int, world: int, total_frames: int, sampler):
    """C5: 512^2 x 32-coil k-space, `total_frames` frames split into contiguous
    slabs over the ranks, each streamed from its rank's pinned buffer (RSS);
    the streamed images are checked against the resident rss_recon process."""
    from paper_1807_11830_b200.sharding import frame_slab
    fb, fe = frame_slab(rank, world, total_frames)
    nfr = fe - fb
    n, nc = C5_NX, C5_NC
    Y5 = h.pinned_empty((n, n, nc, nfr), np.complex64)
    rng = np.random.default_rng(5)
    base = (rng.standard_normal((n, n, nc), dtype=np.float32)
            + 1j * rng.standard_normal((n, n, nc), dtype=np.float32)).astype(np.complex64)
    for i in range(nfr):  # distinct frames at memcpy speed (16 GiB at N=1)
        np.multiply(base, np.float32(1.0 + 0.01 * (fb + i)), out=Y5[..., i])
    R5 = h.pinned_empty((n, n, nfr), np.float32)
    st5 = h.StreamingRecon(s, "rss", n, n, nc, 2)
    st5.run(Y5, R5)
    barrier(world)
    sampler.on()
    s.timer_start()
    reps = 2
    for _ in range(reps):
        st5.run(Y5, R5)
    t5 = reduce_max(s.timer_stop(), world) / reps
    sampler.off()
    # parity: streamed frames (first chunk and the tail) == resident rss_recon
    ok = True
    for f0 in sorted({0, max(0, nfr - 2)}):
        f1 = min(nfr, f0 + 2)
        hk = s.register_data(h.Data([np.asfortranarray(Y5[..., f0:f1])], h.DataKind.KData))
        hr = s.allocate_data([((n, n, f1 - f0), np.float32)], h.DataKind.XData)
        pr = h.Process(s, "rss_recon").set_input(hk).set_output(hr).init()
        pr.launch()
        Rr = s.fetch_data(hr).arrays[0]
        ok &= bool(np.abs(Rr - R5[..., f0:f1]).max() <= 1e-5 * max(np.abs(Rr).max(), 1e-30))
        if f0 == 0:
            td = _device_time(s, pr.launch, 20)
            dev_fps = (f1 - f0) / td
        s.release_data(hk)
        s.release_data(hr)
    ok = reduce_max(0.0 if ok else 1.0, world) == 0.0
    del Y5, R5, st5
    return {"frames_total": total_frames, "ranks": world, "frames_rank0": nfr, "frames_per_s": total_frames / t5,
            "seconds_per_step": t5, "host_link_gbs_rank0": nfr * n * n * nc * 8 / t5 / 1e9,
            "matches_resident": ok, "device_frames_per_s_rank0": dev_fps,
            "device_gbs_rank0": dev_fps * (n * n * nc * 8 + n * n * 4) / 1e9,
            "note": "pinned H2D of 64 MiB/frame (PCIe) dominates; slabs of one volume over the ranks"}


def _device_time(s, fn, reps: int) -> float:
    """Mean device seconds of fn() over reps (CUDA events on the compute stream),
    after 50 untimed calls (the latency-bound configs are host-issue bound, so
    the host side is warmed too)."""
    for _ in range(50):
        fn()
    s.synchronize()
    s.timer_start()
    for _ in range(reps):
        fn()
    return s.timer_stop() / reps


def other_configs(h, s, peak: float):
    """Side measurements for BASELINE.json configs 0, 1, 3 (device resident; C5
    is c5_stream, the headline is config 2 = C3)."""
    rng = np.random.default_rng(99)
    out = {}
    # C1: Negate on one 512x512 float32 image (paper's minimal example)
    x = np.asfortranarray(rng.random((512, 512), dtype=np.float32))
    hx = s.register_data([x])
    hy = s.allocate_data([((512, 512), np.float32)])
    p = h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0})  # LaunchStats sampled
    t = _device_time(s, p.launch, 1000)
    # the same loop with every launch timed (two CUDA event records per launch)
    ps = h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0, "launch_timing": "every"})
    ts = _device_time(s, ps.launch, 1000)
    out["C1_negate_512x512_f32"] = {"us_per_image": t * 1e6, "images_per_s": 1 / t,
                                    "gbs": 2 * x.nbytes / t / 1e9, "frac_of_hbm": 2 * x.nbytes / t / 1e9 / peak,
                                    "us_per_image_every_launch_timed": ts * 1e6,
                                    "note": "2 MB per image: host-issue bound (one Python -> C-ABI -> cudaGraphLaunch per image; "
                                            "device time per launch = host time per launch, profiles/round2_small_configs.md)"}
    # C2: single-frame 256x256, 8 coils, IFFT + RSS
    Y2 = np.asfortranarray((rng.standard_normal((256, 256, 8, 1), dtype=np.float32)
                            + 1j * rng.standard_normal((256, 256, 8, 1), dtype=np.float32)).astype(np.complex64))
    hk = s.register_data(h.Data([Y2], h.DataKind.KData))
    hr = s.allocate_data([((256, 256, 1), np.float32)], h.DataKind.XData)
    p2 = h.Process(s, "rss_recon").set_input(hk).set_output(hr).init()
    t2 = _device_time(s, p2.launch, 1000)
    out["C2_rss_256x256x8x1"] = {"us_per_frame": t2 * 1e6, "frames_per_s": 1 / t2,
                                 "gbs": (Y2.nbytes + 256 * 256 * 4) / t2 / 1e9}
    # C4: iterative loop -- normal operator E^H E (FFT + mask + IFFT + coil combine)
    # on C2 shapes, launched 100x after one init()
    S2 = np.asfortranarray((rng.standard_normal((256, 256, 8), dtype=np.float32) + 0j).astype(np.complex64))
    M2 = np.asfortranarray(Y2[:, :, 0, :])
    mask = np.asfortranarray((rng.random((256, 256)) < 0.33).astype(np.float32))
    hn = s.register_data(h.Data([M2, S2, mask], h.DataKind.XData))
    ho = s.allocate_data([((256, 256, 1), np.complex64)], h.DataKind.XData)
    c4 = {}
    for lt in ("sampled", "every"):
        p4 = h.Process(s, "sense_normal").set_input(hn).set_output(ho).init({"launch_timing": lt})
        p4.launch()
        s.synchronize()
        t0 = time.perf_counter()
        s.timer_start()
        for _ in range(100):
            p4.launch()
        t4 = s.timer_stop() / 100
        wall = (time.perf_counter() - t0) / 100
        st = p4.stats()
        c4[lt] = (t4, wall, st)
    t4, wall, st = c4["sampled"]
    prof4 = p4.profile(reps=20)
    out["C4_normal_op_256x256x8_x100"] = {
        "us_per_launch_device": t4 * 1e6, "us_per_launch_wall": wall * 1e6, "launches": st.launches,
        "init_calls": st.init_calls, "init_ms": st.init_seconds * 1e3,
        "us_per_launch_device_every_launch_timed": c4["every"][0] * 1e6,
        "kernel_us_unlinked": [round(x * 1e6, 2) for x in prof4],
        "kernels_per_launch": len(prof4),
        "note": "one cudaGraphLaunch per launch(); plans/twiddles baked in init(); kernels linked by "
                "programmatic (PDL) graph edges (this process' default); kernel_us_unlinked = per-kernel "
                "times without the graph"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunk", type=int, default=4,
                    help="frames per streamed chunk (e2e); 2-4 measured ~0.5 %% faster than 6-10 "
                         "(shorter pipeline drain, profiles/round2_host_flow.md)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-session-flow", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C1/C2/C4/C5 side measurements")
    ap.add_argument("--c5-frames", type=int, default=256, help="frames of the C5 512^2x32 volume (all ranks)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
