"""Turn ncu raw-page CSVs (gpurun_out/raw_<kernel>.csv) into the committed
profile summaries under profiles/ and the per-element DRAM traffic table that
bench.py reports as roofline.traffic."""
import csv
import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "profiles"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", "")) if vals[i] else 0.0
            out[k] = v * UNIT.get(units[i], 1.0)
    out["kernel"] = vals[hdr.index("Kernel Name")]
    stall = {h.split("stalled_")[-1]: float(vals[i] or 0) for i, h in enumerate(hdr)
             if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")}
    tot = sum(stall.values()) or 1.0
    out["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stall.items(), key=lambda kv: -kv[1])[:8]}
    return out


def main(tag, elements, config="config2"):
    src = ROOT / "gpurun_out"
    traffic_path = OUT / "traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    phase = {"eval_ssim": "eval", "quantize_planar": "quantize", "stats_vec": "stats"}
    summary = {}
    for k, p in phase.items():
        f = src / f"raw_{k}.csv"
        if not f.exists():
            continue
        m = load(f)
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        m["dram_bytes_per_elem"] = dram / elements
        m["achieved_dram_GBps"] = dram / m["gpu__time_duration.sum"] / 1e9
        summary[p] = m
        traffic.setdefault(config, {})[p] = {"dram_bytes_per_elem": m["dram_bytes_per_elem"],
                                              "source": f"profiles/{tag}_ncu_summary.json"}
        for kind in ("details", "source"):
            ext = "txt" if kind == "details" else "csv"
            g = src / f"{kind}_{k}.{ext}"
            if g.exists() and kind == "details":
                shutil.copy(g, OUT / f"{tag}_{k}_details.txt")
    (OUT / f"{tag}_ncu_summary.json").write_text(json.dumps(summary, indent=1))
    traffic_path.write_text(json.dumps(traffic, indent=1))
    lf = src / f"launches_{tag}.csv"
    if lf.exists():
        shutil.copy(lf, OUT / f"{tag}_launches.csv")
    print(json.dumps({p: (round(m["gpu__time_duration.sum"] * 1e3, 3), round(m["dram_bytes_per_elem"], 2),
                          round(m["achieved_dram_GBps"])) for p, m in summary.items()}))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "config2")
