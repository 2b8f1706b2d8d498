import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, vals = rows[0], rows[2]
st = [(float(vals[i] or 0), h.split('stalled_')[-1]) for i, h in enumerate(hdr)
      if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
tot = sum(v for v, _ in st)
print(', '.join(f"{n} {100 * v / tot:.1f}" for v, n in sorted(st, reverse=True)[:10]))
for k in sys.argv[2:]:
    if k in hdr:
        print(k, vals[hdr.index(k)])
