#!/usr/bin/env python
"""Benchmark: cardiac-cine SENSE reconstruction (BASELINE.json configs[2], C3).

One step = one launch of the fused sens_recon process over one 256x256 x 32-coil
x 30-frame cine (k-space + sensitivity maps resident in HBM; 496 MiB of input
per step, larger than the 126 MB L2, so no flush is needed).  Per GPU the
work is fixed (weak scaling): rank r reconstructs its own 30-frame slab.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  `value` = frames/s over all ranks with data
resident (device time, CUDA events on the processes' compute stream, max over
ranks); `e2e` = the same metric through the public streaming API from pinned
host memory with H2D+D2H inside the timed region; `roofline` = the dominant
kernel against MEASURED_PEAKS.json; `cpu_baseline` = the reference library
(oracle/_ref, its own ComputeSession API) on this host's cores.
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
CONFIG = {"workload": "C3 cardiac cine SENSE: 256x256 k-space, 32 coils x 30 frames per GPU, "
                      "IFFT2 + conj-sensitivity coil combine",
          "nx": NX, "ny": NY, "coils": NC, "frames_per_gpu": NF, "dtype_io": "complex64",
          "l2_policy": "inputs (496 MiB/step) larger than L2 (126 MB); no flush"}
# algorithmic bytes (SURVEY.md §8 d): Y 16 MiB + M 0.5 MiB per frame, S 16 MiB once per launch
FRAME_Y = NX * NY * NC * 8
FRAME_M = NX * NY * 8
SMAP = NX * NY * NC * 8


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the GPU is loaded."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(n_gpus: int):
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


def make_inputs(seed: int):
    rng = np.random.default_rng(seed)
    Y = np.empty((NX, NY, NC, NF), np.complex64, order="F")
    for f in range(NF):  # chunked to bound temporaries
        re = rng.standard_normal((NX, NY, NC), dtype=np.float32)
        im = rng.standard_normal((NX, NY, NC), dtype=np.float32)
        Y[..., f] = re + 1j * im
    G = (rng.standard_normal((NX, NY, NC), dtype=np.float32) + 1j * rng.standard_normal((NX, NY, NC), dtype=np.float32))
    S = np.asfortranarray((G / np.sqrt((np.abs(G) ** 2).sum(axis=2, keepdims=True))).astype(np.complex64))
    return Y, S


def cpu_baseline(Y, S, budget_s: float = 12.0):
    """The reference library itself (oracle/_ref) on a bounded sample."""
    from oracle import oracle as o
    sample = 2
    Ys = np.asfortranarray(Y[..., :sample])
    if o.reference_available():
        kind = "reference"
        _, t1, _ = o.ref_recon("sens", Ys, S, reps=1)  # warm-up + estimate
        reps = max(2, min(50, int(budget_s / max(t1, 1e-3))))
        _, mean_s, _ = o.ref_recon("sens", Ys, S, reps=reps)
        cores = o.ref_pool_threads()
    else:  # reference not built on this host: single-thread C port
        kind = "port"
        t0 = time.perf_counter()
        o.sens_recon(Ys, S)
        mean_s = time.perf_counter() - t0
        reps, cores = 1, 1
    return {"value": sample / mean_s, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{sample} of the 30 C3 frames (256x256x32 coils) per launch, {reps} launches, "
                      f"plan baked once; WorkerPool threads = min(hw, 16), host has {os.cpu_count()} cores",
            "seconds_per_frame": mean_s / sample}


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference library driven through its ComputeSession API).  One step =
    register the k-space of a bounded frame sample (the reference's H2D),
    run the SENSE chain, fetch the images (D2H); sensitivity maps and the FFT
    plan are set up once, as on the B200 arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as o
    Y, S = make_inputs(1234)
    sample = 2
    Ys = np.asfortranarray(Y[..., :sample])
    if o.reference_available():
        kind = "reference"
        o.ref_recon_e2e("sens", Ys, S, reps=max(1, min(args.warmup, 2)))
        _, mean_s = o.ref_recon_e2e("sens", Ys, S, reps=args.steps)
        cores = o.ref_pool_threads()
    else:
        kind = "port"
        o.sens_recon(Ys, S)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            o.sens_recon(Ys, S)
        mean_s = (time.perf_counter() - t0) / args.steps
        cores = 1
    value = sample / mean_s
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded N(0,1) k-space)",
            "config": dict(CONFIG, sample_frames_per_step=sample), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{sample} of 30 C3 frames per step: register_data(k-space) + "
                                       f"fft_radix2_pass x18 + complex_element_prod + ximage_sum + fetch_data; "
                                       f"WorkerPool threads = min(hw,16) of {os.cpu_count()} host cores"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    from paper_1807_11830_b200 import hetreco as h

    rank, world, local = dist_setup(args.gpus)
    # host placement: this rank's thread and pinned buffers on its GPU's NUMA node
    # (the CPU-baseline leg below gets the whole host back)
    all_cpus = os.sched_getaffinity(0)
    numa_node = h.bind_to_device_numa(local)
    devs = h.enumerate_devices()
    s = h.ComputeSession(device=devs[local])
    Y, S = make_inputs(1234 + rank)
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((NX, NY, NF), np.complex64)], h.DataKind.XData)
    p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init()

    sampler = ClockSampler(local)
    with sampler:
        # warm-up: W steps, extended to >= 0.5 s of load so clocks settle
        t_end = time.perf_counter() + 0.5
        n = 0
        while n < args.warmup or time.perf_counter() < t_end:
            p.launch()
            n += 1
            if n % 50 == 0:
                s.synchronize()
        s.synchronize()
        barrier(world)
        s.synchronize()
        s.timer_start()
        for _ in range(args.steps):
            p.launch()
        t_dev = s.timer_stop()  # synchronizes the compute stream
        barrier(world)
    t_max = reduce_max(t_dev, world)
    value = NF * world * args.steps / t_max
    clocks = sampler.summary()

    # per-kernel device times (events between kernels on the compute stream)
    prof = p.profile(reps=10)  # [axis1, combine] per frame chunk (one chunk by default)
    k_axis1, k_axis0 = sum(prof[0::2]), sum(prof[1::2])
    bytes_axis1 = 2 * FRAME_Y * NF                 # read Y, write X
    bytes_axis0 = FRAME_Y * NF + SMAP + FRAME_M * NF  # read X + S, write M
    peak, peak_kind = peaks()
    kernels = [
        {"name": "k_fft_strided_ring<256,+1,16,2,32> (axis-1 IFFT, 32-column tiles through a 2-stage cp.async shared-memory ring)", "seconds": k_axis1, "bytes": bytes_axis1,
         "gbs": bytes_axis1 / k_axis1 / 1e9},
        {"name": "k_fft_combine_ss<256,4> (axis-0 IFFT + conj(S) coil combine, map rows staged in smem)",
         "seconds": k_axis0,
         "bytes": bytes_axis0, "gbs": bytes_axis0 / k_axis0 / 1e9},
    ]
    for k in kernels:
        k["frac"] = k["gbs"] / peak
        k["share"] = k["seconds"] / (k_axis1 + k_axis0)
    dom = max(kernels, key=lambda k: k["seconds"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        traffic = tj.get("per_launch_bytes", {}).get("axis1" if dom is kernels[0] else "axis0")
    algo_step = NF * (FRAME_Y + FRAME_M) + SMAP
    roofline = {"bound": "hbm", "achieved": dom["gbs"], "peak": peak, "unit": "GB/s", "frac": dom["frac"],
                "traffic": traffic, "peak_source": peak_kind, "kernel": dom["name"],
                "kernels": kernels,
                "chain_achieved": algo_step / (t_max / args.steps) / 1e9,
                "chain_frac": algo_step / (t_max / args.steps) / 1e9 / peak,
                "algorithmic_bytes_per_step": algo_step}

    # end-to-end through the public streaming API (pinned host memory)
    e2e = None
    if not args.no_e2e:
        Yp = h.pinned_empty((NX, NY, NC, NF), np.complex64)
        Yp[...] = Y
        Mp = h.pinned_empty((NX, NY, NF), np.complex64)
        st = h.StreamingRecon(s, "sense", NX, NY, NC, args.chunk, S)
        for _ in range(max(1, args.warmup // 4)):
            st.run(Yp, Mp)
        barrier(world)
        t0 = time.perf_counter()
        e2e_steps = max(3, min(args.steps, 20))
        for _ in range(e2e_steps):
            st.run(Yp, Mp)
        t_e2e = time.perf_counter() - t0
        barrier(world)
        t_e2e = reduce_max(t_e2e, world)
        e2e = {"value": NF * world * e2e_steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": FRAME_Y * NF,
               "d2h_bytes_per_step": FRAME_M * NF, "steps": e2e_steps, "chunk_frames": args.chunk,
               "host_link_gbs": FRAME_Y * NF * e2e_steps / t_e2e / 1e9,
               "note": "sensitivity maps uploaded once at init (resident), k-space streamed per step"}
        # streamed result equals the resident process output
        M_dev = s.fetch_data(hout).arrays[0]
        e2e["matches_resident"] = bool(np.abs(M_dev - Mp).max() <= 1e-5 * np.abs(M_dev).max())
        # host-link roofline: plain pinned H2D copy of the same bytes on this box
        link = h.CudaBackend(local)
        buf = link.allocate(Yp.nbytes)
        link.upload(buf, 0, Yp.reshape(-1, order="F").view(np.uint8))
        t0 = time.perf_counter()
        for _ in range(3):
            link.upload(buf, 0, Yp.reshape(-1, order="F").view(np.uint8))
        link_gbs = 3 * Yp.nbytes / (time.perf_counter() - t0) / 1e9
        link.release(buf)
        link.close()
        # the reference arm's flow through the operator API with plain
        # (pageable) numpy buffers: register k-space, launch, fetch, release
        # -- per step, as --impl reference does on the CPU
        hs = s.register_data(h.Data([Y], h.DataKind.KData))
        s.release_data(hs)
        Mh = np.empty((NX, NY, NF), np.complex64, order="F")
        smap_h = s.register_data(h.Data([S], h.DataKind.Generic))
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
        s.release_data(smap_h)
        e2e["session_api_pageable"] = {
            "value": NF * world / t_sess, "unit": UNIT, "ms_per_step": t_sess * 1e3,
            "h2d_bytes_per_step": FRAME_Y * NF + SMAP, "d2h_bytes_per_step": FRAME_M * NF,
            "note": "register_data(pageable k-space + maps) + sens_recon launch + fetch_data per step "
                    "(the --impl reference flow); pinned staging ring on the host side"}
        e2e["host_link_peak_gbs"] = link_gbs
        e2e["host_link_frac"] = e2e["host_link_gbs"] / link_gbs
        e2e["host_link_roofline_frames_per_s"] = NF * world * link_gbs * 1e9 / (FRAME_Y * NF)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.sched_setaffinity(0, all_cpus)
        cpu = cpu_baseline(Y, S)

    extras = None
    if rank == 0 and not args.no_extras:
        extras = other_configs(h, s, peak, args.c5_frames)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32 (complex64 I/O, fp32 FFT and coil accumulation)",
                "data": "synthetic (seeded N(0,1) k-space, normalised random sensitivity maps)",
                "config": dict(CONFIG, parallelism=f"frame-slab x{world} (no collective)",
                               host_numa_node_rank0=numa_node),
                "impl": "hetreco-b200",
                "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
                "gpu_launches": 2 * args.steps, "other_configs": extras}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _device_time(s, fn, reps: int) -> float:
    """Mean device seconds of fn() over reps (CUDA events on the compute stream)."""
    for _ in range(3):
        fn()
    s.synchronize()
    s.timer_start()
    for _ in range(reps):
        fn()
    return s.timer_stop() / reps


def other_configs(h, s, peak: float, c5_frames: int):
    """Side measurements for BASELINE.json configs 0, 1, 3, 4 (the headline is
    config 2 = C3).  All device-resident except C5, which streams from pinned
    host memory like the e2e leg."""
    rng = np.random.default_rng(99)
    out = {}
    # C1: Negate on one 512x512 float32 image (paper's minimal example)
    x = np.asfortranarray(rng.random((512, 512), dtype=np.float32))
    hx = s.register_data([x])
    hy = s.allocate_data([((512, 512), np.float32)])
    p = h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0})
    t = _device_time(s, p.launch, 200)
    # the same loop with LaunchStats sampled every 16th launch (a timed CUDA
    # event record costs ~3 us of host time per launch)
    ps = h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0, "launch_timing": "sampled"})
    ts = _device_time(s, ps.launch, 200)
    out["C1_negate_512x512_f32"] = {"us_per_image": t * 1e6, "images_per_s": 1 / t,
                                    "gbs": 2 * x.nbytes / t / 1e9, "frac_of_hbm": 2 * x.nbytes / t / 1e9 / peak,
                                    "us_per_image_sampled_stats": ts * 1e6, "images_per_s_sampled_stats": 1 / ts,
                                    "note": "2 MB per image: launch-latency bound (graph launch ~2 us + per-launch "
                                            "stats events unless launch_timing=sampled)"}
    # C2: single-frame 256x256, 8 coils, IFFT + RSS
    Y2 = np.asfortranarray((rng.standard_normal((256, 256, 8, 1), dtype=np.float32)
                            + 1j * rng.standard_normal((256, 256, 8, 1), dtype=np.float32)).astype(np.complex64))
    hk = s.register_data(h.Data([Y2], h.DataKind.KData))
    hr = s.allocate_data([((256, 256, 1), np.float32)], h.DataKind.XData)
    p2 = h.Process(s, "rss_recon").set_input(hk).set_output(hr).init()
    t2 = _device_time(s, p2.launch, 200)
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
    for lt in ("every", "sampled"):
        p4 = h.Process(s, "sense_normal").set_input(hn).set_output(ho).init({"launch_timing": lt})
        s.synchronize()
        t0 = time.perf_counter()
        s.timer_start()
        for _ in range(100):
            p4.launch()
        t4 = s.timer_stop() / 100
        wall = (time.perf_counter() - t0) / 100
        st = p4.stats()
        c4[lt] = (t4, wall, st)
    t4, wall, st = c4["every"]
    out["C4_normal_op_256x256x8_x100"] = {
        "us_per_launch_device": t4 * 1e6, "us_per_launch_wall": wall * 1e6, "launches": st.launches,
        "init_calls": st.init_calls, "init_ms": st.init_seconds * 1e3,
        "us_per_launch_device_sampled_stats": c4["sampled"][0] * 1e6,
        "kernels_per_launch": 3, "note": "one cudaGraphLaunch per launch(); plans/twiddles baked in init()"}
    # C5: 512x512x32 coils streamed from pinned host memory (RSS), per GPU slab
    if c5_frames > 0:
        Y5 = h.pinned_empty((512, 512, 32, c5_frames), np.complex64)
        for f in range(c5_frames):
            Y5[..., f] = (rng.standard_normal((512, 512, 32), dtype=np.float32)
                          + 1j * rng.standard_normal((512, 512, 32), dtype=np.float32))
        R5 = h.pinned_empty((512, 512, c5_frames), np.float32)
        st5 = h.StreamingRecon(s, "rss", 512, 512, 32, 2)
        st5.run(Y5, R5)
        t0 = time.perf_counter()
        for _ in range(3):
            st5.run(Y5, R5)
        t5 = (time.perf_counter() - t0) / 3
        out["C5_stream_rss_512x512x32"] = {"frames_per_gpu": c5_frames, "frames_per_s": c5_frames / t5,
                                           "host_link_gbs": Y5.nbytes / t5 / 1e9,
                                           "note": "pinned H2D of 64 MiB/frame dominates (PCIe)"}
        hk5 = s.register_data(h.Data([np.asfortranarray(Y5[..., :2])], h.DataKind.KData))
        hr5 = s.allocate_data([((512, 512, 2), np.float32)], h.DataKind.XData)
        p5 = h.Process(s, "rss_recon").set_input(hk5).set_output(hr5).init()
        t5d = _device_time(s, p5.launch, 20)
        out["C5_stream_rss_512x512x32"]["device_frames_per_s"] = 2 / t5d
        out["C5_stream_rss_512x512x32"]["device_gbs"] = 2 * (512 * 512 * 32 * 8 + 512 * 512 * 4) / t5d / 1e9
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunk", type=int, default=6, help="frames per streamed chunk (e2e)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C1/C2/C4/C5 side measurements")
    ap.add_argument("--c5-frames", type=int, default=8, help="frames of the C5 512^2x32 streamed slab")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
