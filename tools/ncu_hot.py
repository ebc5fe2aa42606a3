"""Hot instructions (stall samples) of one kernel in an `ncu --page source --csv` export.

    python tools/ncu_hot.py gpurun_out/src_c5_x.csv [kernel-substring] [n]
"""
import collections
import csv
import sys


def main(path, kname="", n=25):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif r and r[0] == "Address" and cur is not None:
            cur[1] = r
        elif cur is not None and cur[1] is not None and r:
            cur[2].append(r)
    for name, hdr, data in blocks:
        if kname not in name:
            continue
        ia, iss, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        cols = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
        tot = collections.Counter()
        for r in data:
            for c in cols:
                tot[c] += int(r[hdr.index(c)] or 0)
        print(name[:100])
        print("  samples", sum(int(r[iss] or 0) for r in data), "warp-instr", sum(int(r[iex] or 0) for r in data),
              "sass", len(data))
        print("  stalls", tot.most_common(6))
        for i in sorted(range(len(data)), key=lambda i: -int(data[i][iss] or 0))[:n]:
            r = data[i]
            st = sorted(((c, int(r[hdr.index(c)] or 0)) for c in cols), key=lambda x: -x[1])[:2]
            print(f"  {r[iss]:>5} {r[iex]:>9}  {r[ia][:64]:64s} {st}")
        break


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]), *(int(x) for x in sys.argv[3:4]))
