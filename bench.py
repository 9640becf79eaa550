#!/usr/bin/env python
"""Benchmark of the B200 3DGEER render path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE config 2): 1M-Gaussian synthetic scene (synth.random_scene,
seed 0, SH degree 3, scales (0.06k, 0.25k), k = (1e4/N)^1/2), one 1920x1080
BEAP camera with 180 x 101.25 deg FoV.  A step is one full forward frame
(prep -> dup -> sort -> render) of one view.  Under torchrun each rank renders
its own view (rank r: the C2 camera rotated by 2 pi r / N about the scene's y
axis; the scene is replicated, views are independent: weak scaling, no
collective on the data path).

``value`` = frames/s of the whole job with the scene resident in HBM; ``e2e``
= the same metric through the reference-facing drop-in ``renderer.render``
(host float64 arrays in, host float64 arrays out, copies inside the timed
region).  Extra keys: fwd+bwd ms per view (config 3), stage times, per-stage
roofline, the 64-view training step (config 4: fwd -> L1 grad -> bwd per view,
NCCL allreduce of the gradients, Adam), and the CPU baseline (the fp64 C port
of the reference path, oracle/, timed on this host).

``--impl reference`` times that CPU port of the reference path on the same
config (rank 0 only) and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rendered FPS (Mrays/s) at 1080p fisheye, 1M Gaussians; fwd+bwd ms/view"
WORKLOAD = "C2: 1M Gaussians, 1920x1080 BEAP fisheye 180x101.25 deg, forward render"
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # derived: SMs x FP32 lanes x 2 x max clock
SURVEY_K5_FLOPS_PER_PAIR = 46  # K5 algorithmic cost per evaluated pair
SURVEY_K6_FLOPS_PER_PAIR = 128  # K6
SURVEY_K1_BYTES_PER_GAUSSIAN = 340  # K1


def measure_fp32_peak(device: int):
    """FP32 FMA peak measured live on this GPU (geer_measure_fp32_peak: scalar FFMA and packed FFMA2)."""
    import ctypes

    from paper_2505_24053_b200 import _lib

    s, p = ctypes.c_double(0), ctypes.c_double(0)
    _lib.check(_lib.load().geer_measure_fp32_peak(device, ctypes.byref(s), ctypes.byref(p)))
    return {"scalar_ffma": s.value, "packed_ffma2": p.value}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def rank_camera(base, rank, world):
    """C2 camera for rank 0; rank r sees the scene from the C2 pose rotated by 2 pi r / N about y."""
    import workloads as synth
    from paper_2505_24053_b200.scene import Camera

    if rank == 0:
        return base
    ang = 2.0 * math.pi * rank / world
    pos = np.array([-2.0 * math.sin(ang), 0.0, -2.0 * math.cos(ang)])
    rot, t = synth.look_at(pos)
    return Camera(width=base.width, height=base.height, model="beap", rotation=rot, translation=t,
                  fov_x=base.fov_x, fov_y=base.fov_y)


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        # GEER_DIST_BACKEND=gloo runs several ranks on one GPU (host-side test of the multi-rank path)
        backend = os.environ.get("GEER_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend=backend)
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
    return rank, world, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ----------------------------------------------------------------------------- CPU (reference port) timing

def cpu_frame_seconds(scene, cam, threads=None):
    """One full C2 frame of the fp64 C port of the reference path (graph + render)."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    g = O.build_render_graph(scene, cam)
    O.render(scene, cam, None, threads=threads, graph=g)
    return time.perf_counter() - t0


def run_reference(args):
    rank, world, _ = dist_setup(args)
    if rank != 0:
        barrier(world)
        return
    from oracle import oracle as O
    import workloads as synth

    scene = synth.config_scene("C2")
    cam = synth.config_camera("C2")
    O.set_num_threads(os.cpu_count() or 1)  # every host core (torchrun sets OMP_NUM_THREADS=1)
    cores = O.num_threads()
    for _ in range(args.warmup):
        cpu_frame_seconds(scene, cam)
    times = [cpu_frame_seconds(scene, cam) for _ in range(args.steps)]
    total = sum(times)
    fps = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "FPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth.random_scene seed 0)",
        "config": {"workload": WORKLOAD, "gaussians": len(scene), "width": cam.width, "height": cam.height},
        "mrays_per_s": fps * 1920 * 1080 / 1e6,
        "cpu_baseline": {"value": fps, "unit": "FPS", "cores": cores, "kind": "port",
                         "sample": "full C2 frame per step (association + raster), fp64 C port of the reference "
                                   "path (oracle/geer_oracle.c), OpenMP over tiles"},
        "e2e": {"value": fps, "unit": "FPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    barrier(world)


# ----------------------------------------------------------------------------- GPU

def count_launches_per_step(fn):
    """Kernels launched by one call of fn, counted with the CUDA profiler (CUPTI)."""
    import torch

    try:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA" and not e.name.startswith("Memcpy")
                 and not e.name.startswith("Memset") and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
        return len(names), sorted(set(names))
    except Exception as exc:  # profiler unavailable
        return None, [f"profiler unavailable: {exc}"]


def run_ours(args):
    import torch

    rank, world, local = dist_setup(args)
    from paper_2505_24053_b200 import renderer
    import workloads as synth
    from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene

    t_setup = time.perf_counter()
    scene = synth.config_scene("C2", n=args.gaussians)
    base_cam = synth.config_camera("C2")
    cam = rank_camera(base_cam, rank, world)
    cfg = renderer.RenderConfig()
    dscene = DeviceScene.from_scene(scene, device=f"cuda:{local}")
    r = DeviceRenderer(local)
    fp32 = measure_fp32_peak(local)
    fp32_peak = max(fp32.values()) if max(fp32.values()) > 0 else FP32_PEAK_TFLOPS
    h, w = cam.height, cam.width
    out = (torch.empty((h, w, 3), dtype=torch.float32, device="cuda"),
           torch.empty((h, w), dtype=torch.float32, device="cuda"),
           torch.empty((h, w), dtype=torch.int32, device="cuda"))
    stream = torch.cuda.current_stream()

    def step():
        r.forward(dscene, cam, cfg, out=out, sync=False)

    # Frames in flight: each step renders one frame; with --inflight F the steps rotate over F
    # contexts on F streams, so one frame's association overlaps another's raster (a renderer
    # serving many views).  Every frame is complete; the timed region covers all of them.
    nf = max(1, args.inflight)
    rs = [r] + [DeviceRenderer(local) for _ in range(nf - 1)]
    outs = [out] + [tuple(torch.empty_like(t) for t in out) for _ in range(nf - 1)]
    streams = [stream] + [torch.cuda.Stream() for _ in range(nf - 1)]
    counter = [0]

    def step_inflight():
        j = counter[0] % nf
        counter[0] += 1
        with torch.cuda.stream(streams[j]):
            rs[j].forward(dscene, cam, cfg, out=outs[j], sync=False)

    for _ in range(max(args.warmup, 3) * nf):
        step_inflight()
    torch.cuda.synchronize()

    # ---- timed region: K forward frames
    sampler = ClockSampler(local)
    sampler.start()
    t_pre = time.perf_counter()
    while time.perf_counter() - t_pre < 0.3:  # keep the GPU busy while the sampler starts (untimed)
        step()
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s_ in streams[1:]:
        s_.wait_event(ev0)
    for _ in range(args.steps):
        step_inflight()
    for s_ in streams[1:]:
        e_ = torch.cuda.Event()
        e_.record(s_)
        stream.wait_event(e_)
    ev1.record(stream)
    torch.cuda.synchronize()
    for rr_ in rs:  # every timed frame was a complete, error-free frame (device status; no re-run needed)
        rr_.sync()
    barrier(world)
    clocks = sampler.stop()
    ms_local = ev0.elapsed_time(ev1)
    ms_total = allreduce_max(ms_local, world)
    ms_per_step = ms_total / args.steps
    value = world * args.steps / (ms_total / 1e3)

    extra = {}
    # ---- stage times + frame statistics (separate pass; events inside the library)
    r.set_timing(True)
    stage_samples = []
    for _ in range(5):
        step()
        stage_samples.append(r.stats())
    r.set_timing(False)
    st = {k: float(np.median([s[k] for s in stage_samples])) for k in stage_samples[0]}
    n_px = w * h
    pairs = st["evaluated_pairs"]
    peaks = load_peaks()
    stages = {
        "prep": {"ms": st["ms_prep"], "bound": "hbm", "unit": "GB/s",
                 "achieved": len(scene) * SURVEY_K1_BYTES_PER_GAUSSIAN / (st["ms_prep"] * 1e-3) / 1e9},
        "dup": {"ms": st["ms_dup"], "bound": "hbm", "unit": "GB/s",
                "achieved": (len(scene) * (4 * 16 + 24) + st["n_entries"] * 8) / (st["ms_dup"] * 1e-3) / 1e9},
        "sort": {"ms": st["ms_sort"], "bound": "hbm", "unit": "GB/s",
                 "achieved": st["n_entries"] * 32 / (st["ms_sort"] * 1e-3) / 1e9},
        "render": {"ms": st["ms_render"], "bound": "fp32", "unit": "TFLOP/s",
                   "achieved": pairs * SURVEY_K5_FLOPS_PER_PAIR / (st["ms_render"] * 1e-3) / 1e12},
    }
    for k, v in stages.items():
        peak = peaks["hbm_gbs"] if v["bound"] == "hbm" else fp32_peak
        v["peak"] = peak
        v["frac"] = v["achieved"] / peak
    dominant = max(stages, key=lambda k: stages[k]["ms"])
    dv = stages[dominant]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dominant)
    except Exception:
        pass
    ncu_util = None
    try:  # issue-slot and pipe utilisation of the same kernel (ncu --set full, profiles/ncu_utilisation.json)
        with open(os.path.join(ROOT, "profiles", "ncu_utilisation.json")) as f:
            ncu_util = json.load(f).get(dominant)
    except Exception:
        pass
    roofline = {"bound": dv["bound"], "kernel": dominant, "achieved": dv["achieved"], "peak": dv["peak"],
                "unit": dv["unit"], "frac": dv["frac"], "traffic": traffic, "ncu": ncu_util,
                "peak_source": (f"{peaks['source']} MEASURED_PEAKS.json hbm_gbs" if dv["bound"] == "hbm" else
                                f"FP32 FMA peak measured live by geer_measure_fp32_peak {fp32} TFLOP/s "
                                f"(MEASURED_PEAKS.json has no FP32 figure; nominal 148 SM x 128 x 2 x 1.965 GHz "
                                f"= {FP32_PEAK_TFLOPS:.1f})"),
                "work": (f"{pairs:.0f} evaluated pairs x {SURVEY_K5_FLOPS_PER_PAIR} flops (SURVEY 8d)"
                         if dominant == "render" else "algorithmic bytes per SURVEY 8d / DESIGN.md")}
    extra["stages"] = stages
    extra["latency_ms_per_frame"] = st["ms_total"]  # one frame alone on one stream (CUDA events)
    # the same frame captured once into a CUDA graph and replayed (the device path is capturable:
    # no host round trip, the same launches every frame), one frame at a time
    try:
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            r.forward(dscene, cam, cfg, out=out, sync=False)
        stream.wait_stream(cs)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            r.forward(dscene, cam, cfg, out=out, sync=False)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        kg = max(10, args.steps)
        g0.record(stream)
        for _ in range(kg):
            graph.replay()
            g_ = torch.cuda.Event()  # one frame at a time: the next replay waits for this one
            g_.record(stream)
            g_.synchronize()
        g1.record(stream)
        torch.cuda.synchronize()
        r.sync()
        extra["graph_latency_ms_per_frame"] = g0.elapsed_time(g1) / kg
        del graph
        # frames in flight as CUDA graphs: one captured frame per context, replayed round robin on
        # the contexts' streams (every replay runs the whole frame: K1 -> sort -> binning -> raster)
        graphs = []
        for j in range(nf):
            with torch.cuda.stream(streams[j]):
                rs[j].forward(dscene, cam, cfg, out=outs[j], sync=False)
        torch.cuda.synchronize()
        for j in range(nf):
            gj = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gj, stream=streams[j] if j else None):
                rs[j].forward(dscene, cam, cfg, out=outs[j], sync=False)
            graphs.append(gj)
        for j in range(nf):
            with torch.cuda.stream(streams[j]):
                graphs[j].replay()
        torch.cuda.synchronize()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for s_ in streams[1:]:
            s_.wait_event(h0)
        for i in range(args.steps):
            with torch.cuda.stream(streams[i % nf]):
                graphs[i % nf].replay()
        for s_ in streams[1:]:
            e_ = torch.cuda.Event()
            e_.record(s_)
            stream.wait_event(e_)
        h1.record(stream)
        torch.cuda.synchronize()
        for rr_ in rs:
            rr_.sync()
        extra["value_cuda_graphs"] = args.steps / (h0.elapsed_time(h1) / 1e3)
        del graphs
    except Exception as exc:  # noqa: BLE001
        extra["graph_latency_ms_per_frame"] = {"error": repr(exc)}
    extra["frame"] = {"entries": int(st["n_entries"]), "tiles": int(st["n_tiles"]),
                      "work_items": int(st["n_work_items"]), "evaluated_pairs": int(pairs),
                      "pairs_per_pixel": pairs / n_px, "kappa_rechecks": int(st["kappa_rechecks"]),
                      "fixup_pixels": int(st["fixup_pixels"]),
                      "warp_entries": int(st["warp_entries"]),
                      "issued_pairs_over_evaluated": 32 * st["warp_entries"] / max(pairs, 1),
                      "clamped": int(st["clamped"])}

    # ---- fwd + bwd ms per view (config 3)
    dl = torch.randn((h, w, 3), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)) / (h * w)
    grads = dscene.zeros_like_grads()

    def fb():
        r.forward(dscene, cam, cfg, out=out, sync=False)
        r.backward(dl, grads=grads)

    for _ in range(3):
        fb()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    kfb = max(3, min(args.steps, 20))
    e0.record(stream)
    for _ in range(kfb):
        fb()
    e1.record(stream)
    torch.cuda.synchronize()
    fb_ms = allreduce_max(e0.elapsed_time(e1), world) / kfb
    r.set_timing(True)
    fb()
    bst = r.stats()
    r.set_timing(False)
    extra["fwd_bwd_ms_per_view"] = fb_ms
    extra["backward_ms"] = bst["ms_backward"]
    # the same fwd+bwd with views in flight (one view per context/stream, as in the training step)
    fb_grads = [grads] + [dscene.zeros_like_grads() for _ in range(nf - 1)]

    def fb_view(j):
        with torch.cuda.stream(streams[j]):
            rs[j].forward(dscene, cam, cfg, out=outs[j], sync=False)
            rs[j].backward(dl, grads=fb_grads[j])

    for j in range(nf):
        fb_view(j)
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for s_ in streams[1:]:
        s_.wait_event(f0)
    for i in range(kfb):
        fb_view(i % nf)
    for s_ in streams[1:]:
        e_ = torch.cuda.Event()
        e_.record(s_)
        stream.wait_event(e_)
    f1.record(stream)
    torch.cuda.synchronize()
    extra["fwd_bwd_ms_per_view_inflight"] = allreduce_max(f0.elapsed_time(f1), world) / kfb
    extra["views_in_flight"] = nf
    stages["backward"] = {"ms": bst["ms_backward"], "bound": "fp32", "unit": "TFLOP/s",
                          "achieved": pairs * SURVEY_K6_FLOPS_PER_PAIR / (bst["ms_backward"] * 1e-3) / 1e12,
                          "peak": fp32_peak}
    stages["backward"]["frac"] = stages["backward"]["achieved"] / fp32_peak

    # ---- kernel launches per step
    n_launch, names = count_launches_per_step(step)
    gpu_launches = n_launch * args.steps if n_launch is not None else None
    extra["launches_per_step"] = n_launch
    extra["kernels"] = names

    # ---- e2e through the reference-facing host API (host f64 in/out, copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: _pinned_copy(a)
        hscene = type(scene)(pin(scene.means), pin(scene.log_scales), pin(scene.quats), pin(scene.opacity_logits),
                             pin(scene.sh))
        # frames in flight through the public API: one host thread (own context, own stream) per frame
        # in flight, so one frame's PCIe copies overlap another's compute
        import concurrent.futures as cf

        nt = max(1, args.inflight)
        ke = max(3, min(args.steps, 10)) * nt
        pool = cf.ThreadPoolExecutor(max_workers=nt)

        sent = []

        def job(_):
            torch.cuda.set_device(local)
            renderer.render(hscene, cam, cfg, device=local)
            sent.append(renderer.last_h2d_bytes(local))

        list(pool.map(job, range(2 * nt)))  # warm-up: one context per thread
        barrier(world)
        t0 = time.perf_counter()
        list(pool.map(job, range(ke)))
        dt = allreduce_max(time.perf_counter() - t0, world)
        # fwd+bwd end to end: renderer.render_backward (renders, then back-propagates) with a host
        # float64 dL/dimage in and float64 gradients out, the same frames in flight
        dl_host = _pinned_copy(np.random.default_rng(0).standard_normal((int(cam.height), int(cam.width), 3)) * 1e-3)
        sent_b = []

        def job_b(_):
            torch.cuda.set_device(local)
            renderer.render_backward(hscene, cam, dl_host, cfg, device=local)
            sent_b.append(renderer.last_h2d_bytes(local))

        list(pool.map(job_b, range(2 * nt)))
        kb = max(2, min(args.steps, 6)) * nt
        barrier(world)
        t0 = time.perf_counter()
        list(pool.map(job_b, range(kb)))
        dtb = allreduce_max(time.perf_counter() - t0, world)
        pool.shutdown()
        n_grad = len(scene.means) * (3 + 3 + 4 + 1 + scene.sh.shape[1] * 3)
        e2e_fb = {"ms_per_view": 1e3 * dtb / kb, "views_per_s": world * kb / dtb,
                  "h2d_bytes_per_step": int(max(sent_b[-kb:])), "d2h_bytes_per_step": int(4 * n_grad),
                  "api": "paper_2505_24053_b200.renderer.render_backward (geer_render_backward_host)",
                  "note": "fp32 gradients over PCIe, widened to the float64 outputs on host cores (exact)"}
        given = sum(a.nbytes for a in (hscene.means, hscene.log_scales, hscene.quats, hscene.opacity_logits, hscene.sh))
        h2d = max(sent[-ke:])  # what crossed PCIe (fp32 narrowed on host cores + a raw fp64 tail)
        d2h = n_px * (3 * 8 + 8 + 8)
        e2e = {"value": world * ke / dt, "unit": "FPS", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * dt / ke, "api": "paper_2505_24053_b200.renderer.render (geer_render_host)",
               "host_memory": "pinned float64 scene arrays", "frames_in_flight": nt,
               "host_input_bytes_per_step": int(given),
               "host_staging": "float64 -> fp32 on the host worker pool (%d threads), last %.0f%% of the elements sent "
                               "raw and narrowed on the device" % (_lib_host_threads(), 100 * _raw_fraction()),
               "fwd_bwd": e2e_fb}

    # ---- 64-view training step (config 4)
    if not args.no_train:
        try:
            trainer = synth.c4_trainer(scene, n_views=args.train_views, rank=rank, world=world,
                                       device=local, inflight=max(1, args.inflight))
            loss_first = trainer.step(compute_loss=True)  # (untimed warm-up step; loss before any update)
            torch.cuda.synchronize()
            kt = max(2, min(args.steps, 5))
            barrier(world)
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(kt):
                trainer.step()
            t1.record()
            torch.cuda.synchronize()
            tms = allreduce_max(t0.elapsed_time(t1), world) / kt
            loss_after = trainer.step(compute_loss=True)  # (untimed: the loss after 1 + kt Adam steps)
            extra["train_step"] = {"views": args.train_views, "ms_per_step": tms, "views_in_flight": trainer.inflight,
                                   "views_per_s": args.train_views / (tms / 1e3),
                                   "allreduce_bytes": trainer.grad_numel * 4,
                                   "loss_first_step": loss_first, "loss_after_steps": loss_after,
                                   "loss_note": "sum over this rank's views of trainer.loss (trainer.py:114-155)"}
        except Exception as exc:
            extra["train_step"] = {"error": repr(exc)}

    # ---- config 5: 6M Gaussians, 3840x2160 equidistant (KB, k = 0) fisheye, forward (each rank one view)
    if not args.no_c5:
        try:
            extra["c5"] = run_c5(args, rank, world, local)
        except Exception as exc:
            extra["c5"] = {"error": repr(exc)}

    # ---- config 1: 10k Gaussians, 256x256 pinhole (the reference's own CPU-runnable case)
    if not args.no_c1:
        try:
            extra["c1"] = run_c1(args, local)
        except Exception as exc:
            extra["c1"] = {"error": repr(exc)}

    # ---- CPU baseline (rank 0, N=1 only): the fp64 C port of the reference path on this host
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import oracle as O

            O.set_num_threads(os.cpu_count() or 1)
            cpu_s = cpu_frame_seconds(scene, base_cam)
            cpu = {"value": 1.0 / cpu_s, "unit": "FPS", "cores": O.num_threads(), "kind": "port",
                   "sample": "one full C2 frame (association + raster) of the fp64 C port oracle/geer_oracle.c",
                   "seconds": cpu_s}
        except Exception as exc:
            cpu = {"value": None, "unit": "FPS", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
        # the unmodified Python reference (baseline/_ref) on C1, beside the port
        cpu["python_reference_c1"] = time_python_reference_c1()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "FPS", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 raster / f64 association",
            "data": "synthetic (synth.random_scene seed 0, fp32-rounded)",
            "config": {"workload": WORKLOAD, "gaussians": len(scene), "width": w, "height": h},
            "frames_in_flight": nf,
            "fps_single_stream": 1e3 / extra["latency_ms_per_frame"] if extra.get("latency_ms_per_frame") else None,
            "views": "one per rank (rank r: C2 pose rotated 2*pi*r/N about y)",
            "l2": "inputs exceed L2 (scene SoA 236 MB fp32 > 126 MB L2); no explicit flush",
            "mrays_per_s": value * w * h / 1e6,
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": gpu_launches,
            "setup_s": time.perf_counter() - t_setup,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    barrier(world)


def run_c1(args, local):
    """BASELINE config 1 on the GPU: forward FPS (one stream, CUDA events) and fwd+bwd ms per view."""
    import torch

    from paper_2505_24053_b200 import renderer
    import workloads as synth
    from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene

    scene = synth.config_scene("C1")
    cam = synth.config_camera("C1")
    ds = DeviceScene.from_scene(scene, device=f"cuda:{local}")
    cfg = renderer.RenderConfig()
    r = DeviceRenderer(local)
    out = (torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda"),
           torch.empty((cam.height, cam.width), dtype=torch.float32, device="cuda"),
           torch.empty((cam.height, cam.width), dtype=torch.int32, device="cuda"))
    dl = torch.randn((cam.height, cam.width, 3), device="cuda",
                     generator=torch.Generator(device="cuda").manual_seed(1)) / (cam.height * cam.width)
    grads = ds.zeros_like_grads()
    for _ in range(5):
        r.forward(ds, cam, cfg, out=out)
        r.backward(dl, grads=grads)
    torch.cuda.synchronize()
    k = 50
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(k):
        r.forward(ds, cam, cfg, out=out)
    e[1].record()
    for _ in range(k):
        r.forward(ds, cam, cfg, out=out)
        r.backward(dl, grads=grads)
    e[2].record()
    torch.cuda.synchronize()
    fwd_ms = e[0].elapsed_time(e[1]) / k
    return {"workload": "C1: 10k Gaussians, 256x256 pinhole, forward (+ fwd+bwd)", "fps": 1e3 / fwd_ms,
            "ms_per_frame": fwd_ms, "fwd_bwd_ms_per_view": e[1].elapsed_time(e[2]) / k, "steps": k,
            "frames_in_flight": 1}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def time_python_reference_c1():
    """The unmodified reference (raygauss from baseline/_ref, or already importable) on C1: render with
    threads=1 and threads=os.cpu_count(), render_backward with os.cpu_count() (renderer.py:24-54,123,234)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from raygauss import camera as rcam
        from raygauss import renderer as rr
        from raygauss.scene import GaussianScene as RScene
    except Exception as exc:
        return {"unavailable": f"raygauss not importable: {exc}"}
    import workloads as synth

    sc = synth.config_scene("C1")
    cm = synth.config_camera("C1")
    rs = RScene(sc.means, sc.log_scales, sc.quats, sc.opacity_logits, sc.sh)
    rc = rcam.Camera(width=cm.width, height=cm.height, model=cm.model, rotation=cm.rotation,
                     translation=cm.translation, fx=cm.fx, fy=cm.fy, cx=cm.cx, cy=cm.cy)
    ncpu = os.cpu_count() or 1
    res = {"workload": "C1: 10k Gaussians, 256x256 pinhole", "cpu_model": _cpu_model(), "cpu_count": ncpu,
           "note": "unmodified raygauss 0.1.0 (pure Python + numpy); its tile pool is GIL-bound"}
    for th in (1, ncpu):
        t0 = time.perf_counter()
        rr.render(rs, rc, rr.RenderConfig(threads=th))
        res[f"render_s_threads{th}"] = time.perf_counter() - t0
    rng = np.random.default_rng(1)
    dl = rng.standard_normal((cm.height, cm.width, 3)) / (cm.height * cm.width)
    t0 = time.perf_counter()
    rr.render_backward(rs, rc, dl, rr.RenderConfig(threads=ncpu))
    res[f"render_backward_s_threads{ncpu}"] = time.perf_counter() - t0
    res["fps_threads1"] = 1.0 / res["render_s_threads1"]
    return res


def run_c5(args, rank, world, local):
    """BASELINE config 5 forward: K frames timed with CUDA events (max over ranks), stage times, stats."""
    import torch

    from paper_2505_24053_b200 import renderer
    import workloads as synth
    from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene

    scene = synth.config_scene("C5")
    cam = synth.config_camera("C5")
    ds = DeviceScene.from_scene(scene, device=f"cuda:{local}")
    del scene
    cfg = renderer.RenderConfig()
    nf = max(1, args.inflight)
    rs = [DeviceRenderer(local) for _ in range(nf)]
    r = rs[0]
    outs = [(torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda"),
             torch.empty((cam.height, cam.width), dtype=torch.float32, device="cuda"),
             torch.empty((cam.height, cam.width), dtype=torch.int32, device="cuda")) for _ in range(nf)]
    out = outs[0]
    main = torch.cuda.current_stream()
    streams = [main] + [torch.cuda.Stream() for _ in range(nf - 1)]

    def frame(i):
        with torch.cuda.stream(streams[i % nf]):
            rs[i % nf].forward(ds, cam, cfg, out=outs[i % nf], sync=False)

    for i in range(3 * nf):
        frame(i)
    torch.cuda.synchronize()
    k = max(3, min(args.steps, 10))
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s_ in streams[1:]:
        s_.wait_event(e0)
    for i in range(k):
        frame(i)
    for s_ in streams[1:]:
        e_ = torch.cuda.Event()
        e_.record(s_)
        main.wait_event(e_)
    e1.record(main)
    torch.cuda.synchronize()
    ms = allreduce_max(e0.elapsed_time(e1), world) / k
    r.set_timing(True)
    r.forward(ds, cam, cfg, out=out)
    st = r.stats()
    r.set_timing(False)
    return {"workload": "C5: 6M Gaussians, 3840x2160 equidistant KB fisheye (hFoV 180 deg), forward",
            "fps": world * 1e3 / ms, "ms_per_frame": ms, "mrays_per_s": world * 1e3 / ms * cam.width * cam.height / 1e6,
            "steps": k, "frames_in_flight": nf, "latency_ms_per_frame": st["ms_total"],
            "entries": int(st["n_entries"]), "work_items": int(st["n_work_items"]),
            "evaluated_pairs": int(st["evaluated_pairs"]),
            "stages_ms": {key: st["ms_" + key] for key in ("prep", "dup", "sort", "render", "total")}}


def _pinned_copy(a):
    import torch

    a = np.ascontiguousarray(a, dtype=np.float64)
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def _lib_host_threads():
    return int(os.environ.get("GEER_HOST_THREADS", len(os.sched_getaffinity(0))))


def _raw_fraction():
    return float(os.environ.get("GEER_HOST_RAW_FRACTION", "0.1"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    ap.add_argument("--train-views", type=int, default=64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c1", action="store_true")
    ap.add_argument("--inflight", type=int, default=6, help="frames in flight (contexts/streams) for the FPS value")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
