"""Collect the round-2 GPU evidence from gpurun_out/ (tools/r02_final.sh TAG) into profiles/:
launch lists, ncu details / per-opcode tables, bench lines, a per-kernel summary JSON and the
per-element DRAM traffic table bench.py reports as roofline.traffic.

    python tools/make_profiles_r02.py r02f
"""
import collections
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out"
OUT = ROOT / "profiles"
ELEMS = {"5": 96 * 721 * 1440 * 12, "2": 4 * 495 * 128 * 128 * 7}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
KEYS = {
    "duration_s": "gpu__time_duration.sum",
    "dram_read_B": "dram__bytes_read.sum",
    "dram_write_B": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_busy_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smem_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warp_instructions": "smsp__inst_executed.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
PHASE = {"eval_ssim8": "eval", "quantize_planar": "quantize", "stats_vec": "stats", "gram12": "stats",
         "pca_project12": "stats"}


def raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")]}
    for name, key in KEYS.items():
        if key in hdr:
            i = hdr.index(key)
            v = vals[i].replace(",", "")
            out[name] = float(v) * UNIT.get(units[i], 1.0) if v else None
    return out


def stalls(path):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    c = collections.Counter()
    for r in data:
        for i in st:
            c[hdr[i][6:]] += int(r[i] or 0)
    t = sum(c.values()) or 1
    return {k: round(100 * v / t, 1) for k, v in c.most_common(8)}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        n = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[ui], 1e-6)
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    return [{"kernel": n, "launches": a[0], "ms_per_launch": a[1] / a[0], "share": a[1] / tot} for n, a in agg.items()]


def main(tag):
    OUT.mkdir(exist_ok=True)
    summary, traffic = {}, {}
    tp = OUT / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text())
    for cfg, elems in ELEMS.items():
        per_phase = collections.defaultdict(float)
        for f in sorted(SRC.glob(f"raw{cfg}_{tag}_*.csv")):
            k = f.stem.split(f"{tag}_", 1)[1]
            m = raw(f)
            if not m:
                continue
            m["dram_bytes_per_elem"] = (m["dram_read_B"] + m["dram_write_B"]) / elems
            m["thread_instr_per_elem"] = 32 * m["warp_instructions"] / elems
            m["elements"] = elems
            sp = SRC / f"source{cfg}_{tag}_{k}.csv"
            if sp.exists():
                m["stalls_pct"] = stalls(sp)
                ops = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_ops.py"), str(sp), str(elems)],
                                     capture_output=True, text=True).stdout
                (OUT / f"r02_config{cfg}_{k}_opcodes.txt").write_text(ops)
            dp = SRC / f"details{cfg}_{tag}_{k}.txt"
            if dp.exists():
                shutil.copy(dp, OUT / f"r02_config{cfg}_{k}_details.txt")
            summary[f"config{cfg}/{k}"] = m
            per_phase[PHASE.get(k, k)] += m["dram_bytes_per_elem"]
        for ph, v in per_phase.items():
            traffic.setdefault(f"config{cfg}", {})[ph] = {"dram_bytes_per_elem": v,
                                                          "source": "profiles/r02_ncu_summary.json"}
        lp = SRC / f"launches{cfg}_{tag}.csv"
        if lp.exists():
            shutil.copy(lp, OUT / f"r02_config{cfg}_launches.csv")
            summary[f"config{cfg}/launch_list"] = launches(lp)
    (OUT / "r02_ncu_summary.json").write_text(json.dumps(summary, indent=1))
    tp.write_text(json.dumps(traffic, indent=1))
    for c in ("5", "2", "1", "3", "4", "ref"):
        p = SRC / f"bench{c}_{tag}.log"
        if p.exists():
            lines = [ln for ln in p.read_text().splitlines() if ln.startswith("{")]
            if lines:
                (OUT / f"r02_bench_config{c}.json").write_text(lines[-1] + "\n")
    for name, dst in ((f"t_{tag}.log", "r02_gpu_tests.log"), (f"smoke_{tag}.log", "r02_smoke.log"),
                      (f"smi_{tag}.txt", "r02_nvidia_smi.txt"), (f"sass_counts_{tag}.txt", "r02_sass_counts.txt")):
        if (SRC / name).exists():
            shutil.copy(SRC / name, OUT / dst)
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk in ("duration_s", "dram_bytes_per_elem", "issue_busy_pct",
                                                                    "thread_instr_per_elem", "registers")}
                      for k, v in summary.items() if isinstance(v, dict)}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02f")
