"""Print the key numbers of bench JSON lines: python tools/show_bench.py gpurun_out/b5_x.log ..."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        k = {p: round(v["ms"], 2) for p, v in d.get("kernels", {}).items()}
        print(f, d["config"]["workload"][:8], "value", round(d["value"], 2), "ms", round(d["ms_per_step"], 2), k,
              "frac", round(d.get("roofline", {}).get("frac", 0), 3), "psnr", d.get("numerics", {}).get("psnr_db_cube0"),
              "ssim", d.get("numerics", {}).get("ssim_cube0"))
