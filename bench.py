#!/usr/bin/env python
"""Benchmark of the B200 array path on BASELINE.json's headline workload.

Default workload: config 5, the ERA5-shaped cube (float32 [744,721,1440,12]),
the largest single-GPU configuration and the cube `north_star` names for
scaling. One step = per-band statistics + normalisation -> float64 Gram ->
host eigh -> PCA 12->6 projection + per-PC ranges -> 16-bit planar frames ->
decode (dequantise + inverse PCA + de-normalise) -> per-band PSNR + 11x11
Gaussian SSIM, with the cube resident in HBM. Multi-GPU: one process per GPU,
the cube sharded along time; the per-band statistics, the C x C Gram partials,
the PC ranges and the metric sums are combined over NCCL
(paper_2506_19656_b200.dist). `--config 2` runs 64 DeepExtremeCubes
minicubes per GPU (weak scaling, no data-path collective); `--config 1/3/4`
the other BASELINE configurations.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config 5]

With --gpus N > 1 and no torchrun environment the script re-launches itself
under `torch.distributed.run` (one rank per GPU, NCCL, 127.0.0.1).

Metric: Gpixel*band/s (elements of the T*H*W*C cubes per second), whole job.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "Gpixel·band/s encode-prep+decode+PSNR/SSIM"
UNIT = "Gpixel·band/s"
SEED0 = 19656
SHAPE2 = (495, 128, 128, 7)


def _args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--cubes", type=int, default=64, help="config 2: cubes per GPU (64)")
    ap.add_argument("--t", type=int, default=None, help="override T (time-sharded configs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / CPU arm)")
    ap.add_argument("--variant", action="append", default=[], metavar="NAME=VALUE",
                    help="kernel variant for A/B runs (cv_set_variant), e.g. eval_kernel=7")
    return ap.parse_args(argv)


# ------------------------------------------------------------------------------ launcher

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _maybe_spawn(a) -> int | None:
    """--gpus N without a torchrun environment: re-launch under torch.distributed.run."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != a.gpus:
            print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            return 2
        return None
    if a.gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------------------------ workloads

class Workload:
    """Per-rank input, stream spec and algorithmic bytes of one configuration."""

    def __init__(self, cfg: int, rank: int, world: int, cubes: int, t_override=None):
        from paper_2506_19656_b200 import synth

        c = synth.CONFIGS[cfg]
        self.cfg = cfg
        self.name = c["name"]
        self.ssim = c["ssim"]
        self.bit_depth = c["bit_depth"]
        self.n_pcs = c["n_pcs"]
        self.normalize = c.get("normalize", False)
        self.dtype = c["dtype"]
        if cfg == 2:
            self.cubes = cubes
            self.shape = SHAPE2
            self.t0 = 0
            self.t_local = SHAPE2[0]
            self.t_total = SHAPE2[0]
            self.sharded = False
        else:
            self.cubes = 1
            T = t_override or c["shape"][0]
            self.shape = (T,) + tuple(c["shape"][1:])
            base, rem = divmod(T, world)
            self.t0 = rank * base + min(rank, rem)
            self.t_local = base + (1 if rank < rem else 0)
            self.t_total = T
            self.sharded = world > 1
        T, H, W, C = self.shape
        self.elem_rank = self.cubes * self.t_local * H * W * C
        self.elem_total = (self.cubes * world if cfg == 2 else 1) * self.t_total * H * W * C
        s = 2 if self.dtype == "u16" else 4
        b = 1 if self.bit_depth == 8 else 2
        E = self.n_pcs or C
        P = 3 * ((E + 2) // 3)
        R = 3 if self.n_pcs else 2
        # SURVEY.md §8d algorithmic bytes per element: enc = R*s + b*P/C,
        # dec = b*E/C + 4, met = s + 4 (stats / quantise / decode+metrics phases)
        self.alg = {"stats": (R - 1) * s, "quantize": s + b * P / C, "eval": b * E / C + 4 + s + 4}
        self.alg_total = sum(self.alg.values())

    def spec(self):
        from paper_2506_19656_b200 import pipeline

        return pipeline.StreamSpec(self.bit_depth, n_pcs=self.n_pcs, normalize=self.normalize)

    def make_input(self, dev, rank, device_out=None):
        from paper_2506_19656_b200 import synth

        T, H, W, C = self.shape
        if self.cfg == 2:
            return synth.minicube_batch(self.cubes, SEED0 + rank * self.cubes, SHAPE2, device=dev)
        local = (self.t_local, H, W, C)
        if self.cfg == 5:
            return synth.era5(synth.SEEDS[5], local, device=dev, t0=self.t0)
        if self.cfg == 1:
            return synth.minicube(synth.SEEDS[1] + 1000 * rank, local, device=dev)
        if self.cfg == 3:
            return synth.simple_s2(synth.SEEDS[3] + 1000 * rank, local, device=dev)
        return synth.dynamic_earthnet(synth.SEEDS[4] + 1000 * rank, local, device=dev).contiguous()

    def config_json(self, world):
        T, H, W, C = self.shape
        if self.cfg == 2:
            work = (f"config2: {self.cubes} x [495,128,128,7] f32 minicubes per GPU (20% NaN frames, 2% "
                    "NaN pixels), forward fill + stats, 10-bit planar frames (9 planes, repeat pad), "
                    "dequantise, per-band PSNR + 11x11 Gaussian SSIM")
            par = "cube-sharded, one process per GPU, no data-path collective"
        else:
            work = (f"config{self.cfg}: {self.name} [{T},{H},{W},{C}] {self.dtype}, {self.bit_depth}-bit"
                    + (f", PCA {C}->{self.n_pcs}" if self.n_pcs else "")
                    + (" on per-band min/max normalised bands" if self.normalize else "")
                    + (", PSNR + 11x11 Gaussian SSIM" if self.ssim else ", PSNR"))
            par = (f"time-sharded over {world} GPU(s), {self.t_local} frames per GPU; NCCL all-reduce/"
                   "all-gather of band stats, Gram partials, PC ranges, metric sums" if world > 1
                   else "one GPU")
        s = 2 if self.dtype == "u16" else 4
        return {"workload": work, "cubes_per_gpu": self.cubes, "elements_per_gpu": self.elem_rank,
                "bit_depth": self.bit_depth,
                "l2": f"inputs {self.elem_rank * s / 1e9:.1f} GB per GPU >> 126 MB L2 (no flush needed)",
                "parallelism": par}


# ------------------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region through NVML
    (the library behind nvidia-smi) from a background thread. Spawning the
    nvidia-smi CLI while kernels are being launched stalled launches by
    milliseconds (driver lock) and showed up as idle GPU time in short steps."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index: int, period_s: float = 0.05):
        self.idx = gpu_index
        self.period = period_s
        self.samples = []
        self.thread = None
        self.stop_evt = threading.Event()
        self.nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[gpu_index]) if vis and vis.split(",")[0].isdigit() else gpu_index
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml
        except Exception:  # noqa: BLE001 - no NVML: report it, keep benchmarking
            self.nvml = None

    def _run(self):
        p = self.nvml
        while not self.stop_evt.is_set():
            try:
                self.samples.append((p.nvmlDeviceGetClockInfo(self.handle, p.NVML_CLOCK_SM),
                                     p.nvmlDeviceGetCurrentClocksEventReasons(self.handle),
                                     p.nvmlDeviceGetPowerUsage(self.handle) / 1000.0))
            except Exception:  # noqa: BLE001
                pass
            self.stop_evt.wait(self.period)

    def start(self):
        if self.nvml is not None:
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()

    def stop(self) -> dict:
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["NVML unavailable"]}
        self.stop_evt.set()
        self.thread.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        reasons = set()
        for _, mask, _ in self.samples:
            for name, attr in self.REASONS:
                if mask & getattr(self.nvml, attr):
                    reasons.add(name)
        sm = sorted(s[0] for s in self.samples)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(s[2] for s in self.samples), "source": "NVML"}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------------------ CPU arm
#
# The reference's algorithm for this path is cubevid's numpy functions
# (transform.py / cube.py / plan.py / bridge.py) plus the restated metrics
# (SPEC.md:412-436). It is a Python package: there is no C/C++ to build into
# oracle/_ref, and /root/reference is absent on the GPU box, so the CPU arm
# runs the oracle port of those functions (oracle/, pinned to the reference's
# own outputs in tests/golden). Workers are independent processes, one per
# host core; each holds its own sample of the workload (below).

_SAMPLE = {}


def _sample_shape(cfg: int):
    """Bounded per-worker sample of each configuration (full H x W x C)."""
    return {1: (124, 128, 128, 7), 2: (124, 128, 128, 7), 3: (4, 512, 512, 12),
            4: (8, 1024, 1024, 4), 5: (1, 721, 1440, 12)}[cfg]


def _cpu_init(cfg: int, counter):
    import numpy as np  # noqa: F401
    import torch

    torch.set_num_threads(1)
    from paper_2506_19656_b200 import synth

    with counter.get_lock():
        idx = counter.value
        counter.value += 1
    shp = _sample_shape(cfg)
    if cfg in (1, 2):
        x = synth.minicube(SEED0 + idx, shp)
    elif cfg == 3:
        x = synth.simple_s2(synth.SEEDS[3] + idx, shp)
    elif cfg == 4:
        x = synth.dynamic_earthnet(synth.SEEDS[4] + idx, shp)
    else:
        x = synth.era5(synth.SEEDS[5], shp, t0=idx * shp[0])
    _SAMPLE["x"] = x.numpy()
    _SAMPLE["cfg"] = cfg


def _cpu_run(_):
    """The worker's sample through the oracle port: fill -> [normalise -> PCA] ->
    fit_quant -> quantise -> planar frames -> dequantise -> [inverse] -> PSNR [+ SSIM]."""
    import numpy as np

    from oracle import cubevid_oracle as O
    from oracle import metrics_oracle as M
    from paper_2506_19656_b200 import synth

    x = _SAMPLE["x"]
    c = synth.CONFIGS[_SAMPLE["cfg"]]
    t0 = time.perf_counter()
    enc = O.encode_stream(x, c["bit_depth"], n_pcs=c["n_pcs"], normalize=c.get("normalize", False))
    rec = O.decode_stream(enc["frames"], enc, x.shape, c["bit_depth"])
    M.psnr_per_band(enc["filled"], rec)
    if c["ssim"]:
        M.ssim_per_band(enc["filled"], rec)
    return int(np.prod(x.shape)), time.perf_counter() - t0


class CpuArm:
    """One worker process per host core, each with its own sample of the workload."""

    def __init__(self, cfg: int, workers: int):
        import multiprocessing as mp

        self.cfg = cfg
        self.workers = workers
        ctx = mp.get_context("spawn")
        counter = ctx.Value("i", 0)
        self.pool = ctx.Pool(workers, initializer=_cpu_init, initargs=(cfg, counter))
        self.pool.map(_noop, range(workers), chunksize=1)  # wait until every sample exists

    def step(self) -> tuple:
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_run, range(self.workers), chunksize=1)
        dt = time.perf_counter() - t0
        return sum(r[0] for r in res), dt

    def close(self):
        self.pool.close()
        self.pool.join()

    def sample_text(self) -> str:
        T, H, W, C = _sample_shape(self.cfg)
        return (f"{self.workers} worker process(es) x one [{T},{H},{W},{C}] sample of config {self.cfg} "
                "(same generator) per step through the oracle port of cubevid's numpy functions + the "
                "restated metrics (full fill/[normalise+PCA]/quantise/planar/dequantise/[inverse]/"
                "PSNR[/SSIM] pipeline)")


def _noop(_):
    return 0


def _cpu_workers():
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    return max(1, min(n, 32))


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    workers = _cpu_workers()
    arm = CpuArm(a.config, workers)
    for _ in range(a.warmup):
        arm.step()
    tot_e, tot_t = 0, 0.0
    for _ in range(a.steps):
        e, dt = arm.step()
        tot_e += e
        tot_t += dt
    arm.close()
    value = tot_e / tot_t / 1e9
    wl = Workload(a.config, 0, a.gpus, a.cubes, a.t)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * tot_t / a.steps, "higher_is_better": True,
        "scaling": "weak" if a.config == 2 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": wl.config_json(a.gpus),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": arm.sample_text()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU arm

def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_2506_19656_b200 import _lib, pipeline
    from paper_2506_19656_b200.dist import TimeShard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    for kv in a.variant:
        name, value = kv.split("=")
        _lib.set_variant(name, int(value))

    wl = Workload(a.config, rank, world, a.cubes, a.t)
    x = wl.make_input(dev, rank)
    spec = wl.spec()
    shard = TimeShard() if wl.sharded else None
    recon = torch.empty(x.shape, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    wsp = pipeline.Workspace()

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

        enc = pipeline.encode_prep(x, spec, marks=mark, shard=shard, workspace=wsp)
        mark("quantize")
        _, sc = pipeline.decode_eval(enc, x, recon_out=recon, want_ssim=wl.ssim)
        mark("eval")
        if record:
            ev.append(marks)
        return enc, sc

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize(dev)
    # numerics of the warm state (outside the timed region)
    enc, sc = step()
    enc.check()
    rep0 = sc.report()[0]

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    n0 = lib.cv_launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for _ in range(a.steps):
        step(record=True)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    launches = lib.cv_launch_count() - n0
    ms = t_start.elapsed_time(t_end)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / a.steps
    value = wl.elem_total / (ms_step * 1e-3) / 1e9

    # per-phase durations (CUDA events on the launching stream, inside the timed region)
    phase_ms = {p: 0.0 for p in phases}
    for m in ev:
        prev = m["start"]
        for p in phases:
            phase_ms[p] += prev.elapsed_time(m[p])
            prev = m[p]
    for p in phases:
        phase_ms[p] /= len(ev)
    peak, peak_src = _peaks()
    kernels = {}
    for p in phases:
        gbs = wl.elem_rank * wl.alg[p] / (phase_ms[p] * 1e-3) / 1e9 if wl.alg[p] else 0.0
        kernels[p] = {"ms": phase_ms[p], "alg_bytes_per_elem": wl.alg[p], "achieved_gbs": gbs,
                      "frac": gbs / peak, "share": phase_ms[p] / sum(phase_ms.values())}
    dom = max(phases, key=lambda p: phase_ms[p])
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        ent = json.loads(prof.read_text()).get(f"config{a.config}", {}).get(dom)
        if ent:  # ncu dram__bytes_read+write per element (profiles/) x elements per launch
            traffic = ent["dram_bytes_per_elem"] * wl.elem_rank

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": max(3, a.warmup), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if a.config == 2 else "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded generator with the configuration's shapes and statistics, generated "
                "on device)",
        "config": wl.config_json(world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": kernels[dom]["achieved_gbs"],
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": kernels[dom]["achieved_gbs"] / peak, "traffic": traffic,
                     "alg_bytes_per_elem": wl.alg[dom],
                     "pipeline_alg_bytes_per_elem": wl.alg_total,
                     "pipeline_frac": value * 1e9 * wl.alg_total / world / (peak * 1e9)},
        "kernels": kernels,
        "gpu_launches": int(launches),
        "clocks": clk,
        "numerics": {"psnr_db_cube0": rep0["psnr"], "ssim_cube0": rep0.get("ssim"), "bpppb": rep0["bpppb"]},
    }

    # end to end through the public API: pinned host cube -> device -> frames -> host
    # (codec hand-off) -> decoded frames -> device -> recon + metrics -> host
    if not a.no_e2e and not a.profile:
        host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        host.copy_(x)
        shape5 = tuple(x.shape) if x.dim() == 5 else (1,) + tuple(x.shape)
        del recon, x, wsp, enc, sc
        torch.cuda.empty_cache()
        streamer = pipeline.HostStreamer(shape5, host.dtype, spec, chunk=8 if a.config == 2 else 1,
                                         want_ssim=wl.ssim, device=dev, shard=shard)
        host5 = host.view(shape5)
        streamer.run(host5)  # warm-up
        k_e2e = max(1, min(a.steps, 3))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            streamer.run(host5)  # ends with the D2H read of the metric sums (synchronising)
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t0) / k_e2e
        if world > 1:
            tt = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        line["e2e"] = {"value": wl.elem_total / dt / 1e9, "unit": UNIT,
                       "h2d_bytes_per_step": streamer.h2d_bytes, "d2h_bytes_per_step": streamer.d2h_bytes,
                       "ms_per_step": dt * 1e3,
                       "path": "pipeline.HostStreamer: pinned host cube -> encode_prep -> each [b][g] frame "
                               "slice D2H into pinned host memory (codec hand-off) -> decoded frames H2D -> "
                               "decode_eval -> metric sums D2H"
                               + (" (8-cube chunks, copies overlapped with the kernels)" if a.config == 2
                                  else "")}
        del streamer, host, host5
        torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not a.no_cpu_baseline and not a.profile:
        arm = CpuArm(a.config, _cpu_workers())
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
    rc = _maybe_spawn(a)
    if rc is not None:
        return rc
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
