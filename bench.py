#!/usr/bin/env python
"""Benchmark of the B200 array path on BASELINE.json's headline workload.

Workload (BASELINE.json configs[1], "config 2"): per GPU a batch of 64
DeepExtremeCubes-shaped minicubes, float32 [495,128,128,7] with 20% NaN frames
and 2% NaN pixels; one step = forward fill + per-band stats -> 10-bit
quantisation into planar 3-channel frames -> decode (dequantise) -> per-band
PSNR + 11x11 Gaussian SSIM, all cubes, inputs resident in HBM.

Metric: Gpixel*band/s (elements of the T*H*W*C cubes per second), whole job.
Multi-GPU: one process per GPU (torchrun), each rank owns its own 64 cubes
(independent objects: no data-path collective, weak scaling); the step time
is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

SHAPE = (495, 128, 128, 7)
BIT_DEPTH = 10
SEED0 = 19656
METRIC = "Gpixel·band/s encode-prep+decode+PSNR/SSIM"
UNIT = "Gpixel·band/s"
ELEM = SHAPE[0] * SHAPE[1] * SHAPE[2] * SHAPE[3]
# algorithmic bytes per element: s = 4 (f32), b = 2 (10-bit), P = 9, C = E = 7
B_ENC = 2 * 4 + 2 * 9 / 7          # stats pass + quantise pass reads, frame writes
B_DEC = 2 * 7 / 7 + 4              # real planes read, f32 recon write
B_MET = 4 + 4                      # original + recon reads
LAUNCHES_PER_STEP = 6              # stats_reset, stats, stats_finalize, quantize, eval, eval_finalize


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cubes", type=int, default=64, help="cubes per GPU (config 2: 64)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / CPU arm)")
    return ap.parse_args()


# ------------------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.idx)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=5)
        sm, smax, reasons, watts = [], [], set(), []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                watts.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm_sorted = sorted(sm)
        return {"sm_mhz": sm_sorted[len(sm_sorted) // 2], "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(watts)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------------------ CPU arm

def _cpu_worker(args):
    """One cube through the oracle port (numpy), fill -> stats -> quantise ->
    planar frames -> dequantise -> PSNR + SSIM. Returns (elements, seconds)."""
    import numpy as np

    from oracle import cubevid_oracle as O
    from oracle import metrics_oracle as M

    x = args
    t0 = time.perf_counter()
    enc = O.encode_stream(x, BIT_DEPTH)
    rec = O.decode_stream(enc["frames"], enc, x.shape, BIT_DEPTH)
    M.psnr_per_band(enc["filled"], rec)
    M.ssim_per_band(enc["filled"], rec)
    return int(np.prod(x.shape)), time.perf_counter() - t0


class CpuArm:
    """The reference's algorithm (oracle port of cubevid's numpy functions +
    the restated metrics) on the host cores: one worker process per core, each
    processing its own cube sample (cubes are independent)."""

    def __init__(self, workers: int, t_sample: int):
        import multiprocessing as mp

        import torch

        from paper_2506_19656_b200 import synth

        self.workers = workers
        self.t_sample = t_sample
        shape = (t_sample,) + SHAPE[1:]
        self.cubes = [synth.minicube(SEED0 + i, shape, device="cpu").numpy() for i in range(workers)]
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(workers) if workers > 1 else None
        del torch

    def step(self) -> tuple:
        t0 = time.perf_counter()
        if self.pool is None:
            res = [_cpu_worker(self.cubes[0])]
        else:
            res = self.pool.map(_cpu_worker, self.cubes, chunksize=1)
        dt = time.perf_counter() - t0
        return sum(r[0] for r in res), dt

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()

    def sample_text(self) -> str:
        return (f"{self.workers} worker process(es) x one [{self.t_sample},128,128,7] f32 minicube "
                f"(config-2 generator, {self.t_sample}/495 time steps) per step, full pipeline "
                "fill/stats/10-bit quantise/planar/dequantise/PSNR/SSIM-11x11")


def _cpu_workers():
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    return max(1, min(n, 32))


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    workers = _cpu_workers()
    arm = CpuArm(workers, t_sample=124)
    for _ in range(a.warmup):
        arm.step()
    tot_e, tot_t = 0, 0.0
    for _ in range(a.steps):
        e, dt = arm.step()
        tot_e += e
        tot_t += dt
    arm.close()
    value = tot_e / tot_t / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * tot_t / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config(a.cubes),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": arm.sample_text()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(cubes):
    return {
        "workload": f"config2: {cubes} x [495,128,128,7] f32 minicubes per GPU (20% NaN frames, 2% NaN "
                    "pixels), forward fill + stats, 10-bit planar frames (9 planes, repeat pad), "
                    "dequantise, per-band PSNR + 11x11 Gaussian SSIM",
        "cubes_per_gpu": cubes,
        "elements_per_gpu": cubes * ELEM,
        "bit_depth": BIT_DEPTH,
        "l2": "inputs 14.5 GB per GPU >> 126 MB L2 (no flush needed)",
        "parallelism": "cube-sharded, one process per GPU, no data-path collective",
    }


# ------------------------------------------------------------------------------ GPU arm

def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_2506_19656_b200 import _lib, pipeline, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()

    B = a.cubes
    x = synth.minicube_batch(B, SEED0 + rank * B, SHAPE, device=dev)
    spec = pipeline.StreamSpec(BIT_DEPTH)
    recon = torch.empty(x.shape, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    phases = ("stats", "quantize", "eval")
    ev = []

    def step(record=False):
        marks = {}
        if record:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            marks["start"] = e0

        def mark(label):
            if record:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks[label] = e

        enc = pipeline.encode_prep(x, spec, marks=mark)
        mark("quantize")
        _, sc = pipeline.decode_eval(enc, x, recon_out=recon)
        mark("eval")
        if record:
            ev.append(marks)
        return enc, sc

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    # numerics sanity of the warm state (outside the timed region)
    enc, sc = step()
    enc.check()
    rep0 = sc.report()[0]

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for _ in range(a.steps):
        step(record=True)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    ms = t_start.elapsed_time(t_end)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / a.steps
    total_elem = world * B * ELEM
    value = total_elem / (ms_step * 1e-3) / 1e9

    # per-phase durations (CUDA events on the launching stream, inside the timed region)
    phase_ms = {p: 0.0 for p in phases}
    for m in ev:
        prev = m["start"]
        for p in phases:
            phase_ms[p] += prev.elapsed_time(m[p])
            prev = m[p]
    for p in phases:
        phase_ms[p] /= len(ev)
    per_rank_elem = B * ELEM
    alg = {"stats": 4.0, "quantize": 4.0 + 2 * 9 / 7, "eval": B_DEC + B_MET}
    peak, peak_src = _peaks()
    kernels = {}
    for p in phases:
        gbs = per_rank_elem * alg[p] / (phase_ms[p] * 1e-3) / 1e9
        kernels[p] = {"ms": phase_ms[p], "alg_bytes_per_elem": alg[p], "achieved_gbs": gbs,
                      "frac": gbs / peak, "share": phase_ms[p] / sum(phase_ms.values())}
    dom = max(phases, key=lambda p: phase_ms[p])
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(dom)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded config-2 generator on device: smooth fields + annual cycle + AR(1), "
                "NaN clouds)",
        "config": _config(B),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": kernels[dom]["achieved_gbs"],
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": kernels[dom]["achieved_gbs"] / peak, "traffic": traffic,
                     "alg_bytes_per_elem": alg[dom],
                     "pipeline_frac": value * 1e9 * (B_ENC + B_DEC + B_MET) / world / (peak * 1e9)},
        "kernels": kernels,
        "gpu_launches": LAUNCHES_PER_STEP * a.steps,
        "clocks": clk,
        "numerics": {"psnr_db_cube0": rep0["psnr"], "ssim_cube0": rep0["ssim"], "bpppb": rep0["bpppb"]},
    }

    # end-to-end through the public API with pinned host buffers
    if not a.no_e2e and not a.profile:
        host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        host.copy_(x)
        del recon
        streamer = pipeline.HostStreamer(tuple(x.shape), x.dtype, spec, chunk=8, device=dev)
        del x
        torch.cuda.empty_cache()
        streamer.run(host)  # warm-up
        k_e2e = max(1, min(a.steps, 3))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            streamer.run(host)  # ends with the D2H read of the metric sums (synchronising)
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t0) / k_e2e
        if world > 1:
            tt = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        line["e2e"] = {"value": total_elem / dt / 1e9, "unit": UNIT,
                       "h2d_bytes_per_step": streamer.h2d_bytes, "d2h_bytes_per_step": streamer.d2h_bytes,
                       "ms_per_step": dt * 1e3, "path": "pipeline.HostStreamer (pinned host, 8-cube "
                       "chunks, copy stream overlapped with the kernels)"}

    if rank == 0 and world == 1 and not a.no_cpu_baseline and not a.profile:
        arm = CpuArm(_cpu_workers(), t_sample=124)
        e, dt = arm.step()
        arm.close()
        line["cpu_baseline"] = {"value": e / dt / 1e9, "unit": UNIT, "cores": arm.workers, "kind": "port",
                                "sample": arm.sample_text(), "seconds": dt}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
