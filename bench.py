"""bench.py -- exact squared-EDT throughput on B200 (BASELINE.json metric).

Workload (config.workload): BASELINE.json configs[1] ("c2"): one 4096x4096
uint8 image of 200 seeded discs (radii 8..64), exact squared EDT in BOTH
directions (background->object = edt(img), object->background =
edt(img.inverted())) as int32 plus float32 distances.  A step = one pass of
the hot path over that image.  Under torchrun (N>1) every rank transforms its
own replica (seed + rank): C2 is a single image the spec does not shard, so
N>1 is replicas only ("scaling": "weak"), and the value is the whole-job
pixel rate (N * pixels / max-over-ranks time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c1|c2|c3|c4|c5]   (default c2; others for study)

Timing: W >= 3 untimed warm-ups; every timed step is bracketed by CUDA events
on the launching stream, with a 256 MiB L2 flush (> 126 MB L2) BETWEEN steps
outside the events; barrier + synchronize on both sides of the timed region;
max over ranks.  The dominant kernel (the row pass) is timed by events the C
ABI records on the same stream (dfc_set_profile_events).  Clocks and
throttle reasons are sampled with NVML during the timed region.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified proj/core sources compiled in this repo) on the host cores, same
config/metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback

CONFIGS = {
    "c1": dict(desc="c1: 600x500 uint8 Bernoulli p=0.01 (reference generator), exact squared EDT "
                    "int32 + float32 distances", bytes_alg=9, bytes_kernel=8 + 0.25),  # k_rows_anc: outputs + band masks/carries
    "c2": dict(desc="c2: 4096x4096 uint8, 200 seeded discs (r 8..64), exact squared EDT both "
                    "polarities int32 + float32 distances", bytes_alg=17,
               bytes_kernel=16 + 0.375),  # k_rows_anc: 2 x 8 B outputs + band masks (shared) and carries / 32 rows
    "c3": dict(desc="c3: 1024 images 1024x1024 uint8, 30 seeded points each, exact squared EDT "
                    "int32 + int32 Voronoi labels", bytes_alg=9, bytes_kernel=8),  # point planes: no nr plane
    "c4": dict(desc="c4: 8192x8192 uint8, 2000 seeded discs/rectangles, city-block + chessboard + "
                    "chamfer-3-4 int32", bytes_alg=13, bytes_kernel=2 + 12),
    "c5": dict(desc="c5: 32768x32768 uint8, Bernoulli 1e-4 in 256 of 1024 tiles, exact squared "
                    "EDT int32", bytes_alg=5, bytes_kernel=2 + 4),
}


# what the timed "row pass" of each config runs (the default per-plane dispatch)
ROW_KERNELS = {
    "c1": "row pass (k_rows_anc: the plane is neither dense nor sparse)",
    "c2": "row pass (k_rows_anc, both planes)",
    "c3": "row pass (k_rows_pts: every image is a point plane, <= 32 object pixels)",
    "c4": "k_band_* + k_raster_anc (whole step)",
    "c5": "row pass (k_rows_lr: a sparse plane)",
}


def traffic_for(cfg):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(cfg)
        return (t["dram_bytes_per_launch"], t["source"]) if t else (None, None)
    except Exception:
        return None, None


def peaks():
    try:
        with open(MEASURED) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index):
        self.ok = False
        self.samples, self.reasons = [], set()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for bit, name in self.REASONS.items():
            if r & bit and bit != 0x1:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()
            return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.samples)}
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}


def make_input(cfg, rank):
    from paper_2106_03503_b200 import workloads
    seed = workloads.SEEDS[cfg] + rank
    return workloads.config(cfg, seed=seed), seed


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2106_03503_b200 as dfc

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = args.config
    sharded_mode = world > 1 and cfg in ("c3", "c5")
    img_np, seed = make_input(cfg, 0 if sharded_mode else rank)
    job_px = img_np.size if sharded_mode else img_np.size * world   # pixels the whole job does per step
    if sharded_mode and cfg == "c3":      # per-image shards, no collective
        from paper_2106_03503_b200.sharded import shard_range
        lo, hi = shard_range(img_np.shape[0], rank, world)
        img_np = np.ascontiguousarray(img_np[lo:hi])
    H5 = W5 = None
    if sharded_mode and cfg == "c5":      # column stripes -> NCCL all-to-all -> row stripes
        H5, W5 = img_np.shape
        Ws = W5 // world
        img_np = np.ascontiguousarray(img_np[:, rank * Ws:(rank + 1) * Ws])
    img = torch.from_numpy(img_np).to(dev)
    npx = img_np.size
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # preallocated outputs (a step writes them; no allocation in the timed region)
    if cfg == "c2":
        out = {k: torch.empty(img_np.shape, dtype=dt, device=dev)
               for k, dt in (("sqdist_bg", torch.int32), ("dist_bg", torch.float32),
                             ("sqdist_obj", torch.int32), ("dist_obj", torch.float32))}
        step = lambda: dfc.edt_dual(img, out=out)
    elif sharded_mode and cfg == "c5":
        from paper_2106_03503_b200 import sharded
        out = {}
        step = lambda: sharded.edt_column_striped(img, H5, W5, rank, world)
    elif cfg == "c1" or cfg == "c5":
        out = {"sqdist": torch.empty(img_np.shape, dtype=torch.int32, device=dev)}
        if cfg == "c1":
            out["dist"] = torch.empty(img_np.shape, dtype=torch.float32, device=dev)
        step = lambda: dfc.edt(img, dist=cfg == "c1", out=out)
    elif cfg == "c3":
        out = {k: torch.empty(img_np.shape, dtype=torch.int32, device=dev) for k in ("sqdist", "label")}
        step = lambda: dfc.edt_batched(img, dist=False, label=True, out=out)
    else:  # c4
        out = {k: torch.empty(img_np.shape, dtype=torch.int32, device=dev)
               for k in ("cityblock", "chessboard", "chamfer34")}
        step = lambda: dfc.raster(img, out=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = dfc.last_launch_count()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for tup in ev:  # torch creates the cudaEvent_t lazily at the first record
        for e in tup:
            e.record(stream)
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        flush.fill_(k & 0xFF)  # evict L2 between timed steps (outside the events)
        e0, e1, e2, e3 = ev[k]
        if cfg != "c4":
            dfc.set_profile_events(None, e1, e2)
        e0.record(stream)
        step()
        e3.record(stream)
    torch.cuda.synchronize()
    dfc.set_profile_events(None, None, None)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(d) for a, _, _, d in ev]
    total_ms = float(sum(step_ms))
    if cfg != "c4":
        row_ms = float(np.mean([b.elapsed_time(c) for _, b, c, _ in ev]))
    else:
        row_ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([total_ms, row_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, row_ms = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    value = job_px * args.steps / (total_ms * 1e-3) / 1e6

    # ---- e2e through the public API with HOST buffers (pinned), copies timed ----
    # Two streams, each with its own device input/outputs and pinned host
    # outputs: step k's device->host copies overlap step k+1's upload and
    # compute (a streaming caller's pipeline).  Every step still copies its
    # input in and all its result maps out inside the timed region.
    host_in = torch.from_numpy(img_np).pin_memory()
    streams = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
    bufs = []
    for _ in range(2):
        o = {k: torch.empty_like(v) for k, v in out.items()}
        bufs.append({"dev_in": torch.empty_like(img), "out": o,
                     "host_out": {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in o.items()},
                     "extra": {}})

    def e2e_step(k):
        bf = bufs[k & 1]
        with torch.cuda.stream(streams[k & 1]):
            bf["dev_in"].copy_(host_in, non_blocking=True)
            x = bf["dev_in"]
            o = bf["out"]
            if sharded_mode and cfg == "c5":
                _, _, sq = sharded.edt_column_striped(x, H5, W5, rank, world)
                if "sq" not in bf["extra"]:
                    bf["extra"]["sq"] = torch.empty(sq.shape, dtype=sq.dtype).pin_memory()
                bf["extra"]["sq"].copy_(sq, non_blocking=True)
                return
            if cfg == "c2":
                dfc.edt_dual(x, out=o)
            elif cfg in ("c1", "c5"):
                dfc.edt(x, dist=cfg == "c1", out=o)
            elif cfg == "c3":
                dfc.edt_batched(x, dist=False, label=True, out=o)
            else:
                dfc.raster(x, out=o)
            for k2, v in o.items():
                bf["host_out"][k2].copy_(v, non_blocking=True)

    e2e_steps = max(4, min(args.steps, 10))
    for k in range(2):
        e2e_step(k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    a.record(stream)
    for s_ in streams:
        s_.wait_event(a)
    for k in range(e2e_steps):
        e2e_step(k)
    for s_ in streams:
        stream.wait_stream(s_)
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    host_out = bufs[0]["host_out"]
    e2e_host_out = bufs[0]["extra"]
    h2d = int(host_in.numel() * host_in.element_size())
    d2h = int(sum(v.numel() * v.element_size() for v in host_out.values())) + \
        int(sum(v.numel() * v.element_size() for v in e2e_host_out.values()))

    if rank != 0:
        return None
    peak, peak_src = peaks()
    c = CONFIGS[cfg]
    kernel_bytes = c["bytes_kernel"] * (npx if not (sharded_mode and cfg == "c5") else H5 * W5 // world)
    achieved = kernel_bytes / (row_ms * 1e-3) / 1e9
    step_achieved = c["bytes_alg"] * job_px / world / (ms_per_step * 1e-3) / 1e9
    line = {
        "metric": "exact squared-EDT Mpixel/s (bit-exact)" if cfg != "c4" else "raster DT Mpixel/s (bit-exact)",
        "value": round(value, 1),
        "unit": "Mpixel/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True,
        "scaling": "strong" if sharded_mode else "weak",
        "vs_baseline": None,
        "dtype": "u8->int32" + ("+f32" if cfg in ("c1", "c2") else ""),
        "data": "synthetic (seeded stand-in, SURVEY.md 8(d))",
        "config": {"workload": c["desc"], "seed": seed, "pixels_per_gpu_step": npx,
                   "parallelism": ("single GPU" if world == 1 else
                                   f"replicas x{world}" if not sharded_mode else
                                   f"per-image shards x{world}" if cfg == "c3" else
                                   f"column stripes -> NCCL all-to-all -> row stripes x{world}"),
                   "l2": "256 MiB flush between timed steps (outside the events)"},
        "roofline": {
            "bound": "hbm", "kernel": ROW_KERNELS.get(cfg, "row pass (the row envelope)"),
            "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic_for(cfg)[0],
            "traffic_source": traffic_for(cfg)[1], "algorithmic_bytes_per_launch": kernel_bytes,
            "bytes_per_px": c["bytes_kernel"], "kernel_ms": round(row_ms, 5),
            "step": {"bytes_alg_per_px": c["bytes_alg"], "achieved": round(step_achieved, 1),
                     "frac": round(step_achieved / peak, 4)},
        },
        "e2e": {"value": round(job_px / (e2e_ms * 1e-3) / 1e6, 1), "unit": "Mpixel/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "clocks": clk,
        "gpu_launches": launches_per_step * args.steps,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, img_np)
    return line


# ------------------------------------------------------------- CPU reference
def _ref_step(cfg, img, threads):
    """One bounded sample of the workload on the reference CPU path; returns
    (pixels, seconds) measured by the reference shim's steady_clock."""
    import oracle
    if cfg in ("c1", "c2", "c5"):
        _, ns = oracle.ref_edt(img, threads=threads, want_time=True)
        t = ns
        if cfg == "c2":
            _, ns2 = oracle.ref_edt((img == 0).astype(np.uint8), threads=threads, want_time=True)
            t += ns2
        return img.size, t * 1e-9
    if cfg == "c3":
        sub = np.ascontiguousarray(img[:4])
        import ctypes as C
        ns = C.c_double(0)
        oracle.ref.dfref_edt_labels_batch(sub, sub.shape[0], sub.shape[1], sub.shape[2], threads,
                                          None, None, C.byref(ns))
        return sub.size, ns.value * 1e-9
    # c4: cityblock_sequential + chamfer34 (single-threaded by API) + chessboard restatement
    _, t1 = oracle.ref_propagation(img, 0, want_time=True)
    _, t2 = oracle.ref_propagation(img, 2, want_time=True)
    t0 = time.perf_counter()
    oracle.chessboard(img)
    return img.size, (t1 + t2) * 1e-9 + (time.perf_counter() - t0)


def cpu_baseline(cfg, img):
    import oracle
    threads = os.cpu_count() or 1
    if not oracle.ref_available():
        return {"value": None, "unit": "Mpixel/s", "cores": threads, "kind": "reference",
                "sample": "oracle/_ref/libdfref.so missing"}
    sample_img = img
    note = "full image"
    if cfg == "c5":  # 1 Gpixel is ~1 min: bound the sample to a 8192x8192 crop
        sample_img = np.ascontiguousarray(img[:8192, :8192])
        note = "top-left 8192x8192 crop of the c5 image"
    if cfg == "c3":
        note = "4 of the 1024 images (edt + voronoi_labels each)"
    px, sec = _ref_step(cfg, sample_img, threads)
    if cfg == "c2":
        note = "full image, edt(img) + edt(img.inverted())"
    return {"value": round(px / sec / 1e6, 3), "unit": "Mpixel/s", "cores": threads,
            "kind": "reference", "sample": note + f", threads={threads}", "seconds": round(sec, 3)}


def run_reference(args, rank):
    if rank != 0:
        return None
    import oracle
    cfg = args.config
    img, seed = make_input(cfg, 0)
    threads = os.cpu_count() or 1
    if not oracle.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libdfref.so not built"}
    if cfg == "c5":
        img = np.ascontiguousarray(img[:8192, :8192])
    for _ in range(min(args.warmup, 1)):
        _ref_step(cfg, img, threads)
    tot_px, tot_s = 0, 0.0
    for _ in range(args.steps):
        px, s = _ref_step(cfg, img, threads)
        tot_px += px
        tot_s += s
    value = tot_px / tot_s / 1e6
    c = CONFIGS[cfg]
    sample = {"c2": "full 4096x4096 image, edt(img) + edt(img.inverted())",
              "c1": "full image", "c3": "4 of the 1024 images per step",
              "c4": "full image: cityblock_sequential + chamfer34 + chessboard restatement",
              "c5": "top-left 8192x8192 crop"}[cfg]
    return {
        "impl": "reference", "metric": "exact squared-EDT Mpixel/s (bit-exact)", "value": round(value, 3),
        "unit": "Mpixel/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot_s / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8->uint64", "data": "synthetic",
        "config": {"workload": c["desc"], "seed": seed, "parallelism": f"std::jthread x{threads}"},
        "cpu_baseline": {"value": round(value, 3), "unit": "Mpixel/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    p.add_argument("--no-cpu-baseline", action="store_true")
    args = p.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl")
        line = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
