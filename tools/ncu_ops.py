"""Per-opcode summary of an ncu --page source --csv export (SASS view):
executed thread-instructions per element and share of warp-stall samples."""
import collections
import csv
import sys


def main(path, elements):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    iS, iE = hdr.index("Source"), hdr.index("Thread Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    cnt, st = collections.Counter(), collections.Counter()
    for r in data:
        op = r[iS].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        o = o.split(".")[0]
        cnt[o] += int(r[iE] or 0)
        st[o] += int(r[iW] or 0)
    tot, tots = sum(cnt.values()), sum(st.values()) or 1
    print(f"total {tot / elements:.1f} thread-instr/elem")
    for o, e in cnt.most_common(28):
        print(f"{o:12s} {e / elements:7.2f}  stall {100 * st[o] / tots:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
