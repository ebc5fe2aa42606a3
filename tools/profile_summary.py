"""Summarise an ncu launch list + full-set raw export of one step into profiles/.

    python tools/profile_summary.py TAG CFG   (reads gpurun_out/launches_CFG_TAG.csv, raw_CFG_TAG.csv)

Writes profiles/ncu_CFG_TAG.md (step-kernel shares from the launch list, full-set
metrics per kernel) and profiles/ncu_traffic.json (DRAM bytes per launch of each
kernel class, used by bench.py's roofline 'traffic').
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SETUP = ("factor_kernel", "material_pass", "abc_kernel", "pec_zero", "minmax", "fill_kernel", "check_positive")


def kclass(name):
    if "rhs_kernel" in name:
        return "rhs_e" if "rhs_kernel<2, 0," in name or ", 0, " in name.split("rhs_kernel<")[1][:6] else "rhs_h"
    if "sweep_kernel" in name:
        mode = name.split("sweep_kernel<")[1].split(">")[0].split(",")[1].strip()
        return {"0": "sweep_mass", "1": "sweep_mod", "2": "sweep_der"}[mode]
    return "other"


def to_ms(v, u):
    v = float(v.replace(",", ""))
    return {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6) * v


def main(tag, cfg):
    go = os.path.join(ROOT, "gpurun_out")
    rows = list(csv.reader(open(os.path.join(go, f"launches_{cfg}_{tag}.csv"))))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[h], rows[h + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    step = [(r[ik], to_ms(r[iv], r[iu])) for r in data if not any(s in r[ik] for s in SETUP)]
    tot = sum(ms for _, ms in step)
    per = {}
    for name, ms in step:
        c = kclass(name)
        per.setdefault(c, [0, 0.0])
        per[c][0] += 1
        per[c][1] += ms
    out = [f"# ncu evidence, {cfg}, tag {tag}", "",
           "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` over one step of "
           "`tools/profile_step.py --config %s --steps 1` (cold-cache, serialised: compare shares, not absolutes)." % cfg,
           "", f"Step kernels: {len(step)} launches, {tot:.3f} ms total.", "",
           "| class | launches | ms | share |", "|---|---|---|---|"]
    for c, (n, ms) in sorted(per.items(), key=lambda x: -x[1][1]):
        out.append(f"| {c} | {n} | {ms:.3f} | {ms / tot * 100:.1f}% |")
    raw = list(csv.reader(open(os.path.join(go, f"raw_{cfg}_{tag}.csv"))))
    rh, ru, rd = raw[0], raw[1], raw[2:]
    ix = {k: i for i, k in enumerate(rh)}
    keys = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
            ("launch__registers_per_thread", "regs"), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
            ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %")]
    out += ["", "Full sets (`ncu --set full --clock-control none --import-source on`), first launches of the step:", "",
            "| kernel | " + " | ".join(n for _, n in keys) + " |", "|---" * (len(keys) + 1) + "|"]
    traffic = {}
    for r in rd:
        name = r[ix["Kernel Name"]]
        vals = []
        for k, _ in keys:
            v, u = r[ix[k]], ru[ix[k]]
            vals.append(f"{v} {u}".strip())
        out.append(f"| `{name.split('(')[0].replace('void ', '')}` | " + " | ".join(vals) + " |")
        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = sum(float(r[ix[k]].replace(",", "")) * mul.get(ru[ix[k]], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        traffic.setdefault(kclass(name), []).append(b)
    # one launch per RHS component (rounds before r1e: interior-tile + boundary-tile
    # launches, captured as two kernels of the same class; pass --split-rhs for those)
    split = "--split-rhs" in sys.argv
    bpl = {}
    for c, v in traffic.items():
        bpl[c] = sum(v) / (len(v) / 2 if split and c in ("rhs_e", "rhs_h") else len(v))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"ncu_{cfg}_{tag}.md"), "w").write("\n".join(out) + "\n")
    json.dump({"config": cfg, "tag": tag, "bytes_per_launch": bpl,
               "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full capture "
                       "(rhs_e/rhs_h: one launch per component)"},
              open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(out))
    print(bpl)


if __name__ == "__main__":
    main(*sys.argv[1:3])
