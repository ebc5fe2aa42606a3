"""SASS opcode mix (executed warp instructions) of the first kernel in an `ncu --page source --csv` export.

    python tools/ncu_mix.py gpurun_out/src_x.csv [n]
"""
import collections
import csv
import sys


def main(path, n=25):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "Address":
            if hdr is not None:
                break
            hdr = r
        elif hdr is not None and r:
            data.append(r)
    ia, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    c = collections.Counter()
    for r in data:
        op = r[ia].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += int(r[iex] or 0)
    tot = sum(c.values())
    print(f"total {tot / 1e6:.1f}M warp instructions")
    for o, k in c.most_common(int(n)):
        print(f"  {o:10s} {k / 1e6:9.1f}M {k / tot * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], *sys.argv[2:3])
