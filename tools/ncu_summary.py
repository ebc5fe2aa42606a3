"""Summarise an ncu report (per kernel launch): duration, DRAM bytes, throughput, stalls.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_lsb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_bar",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_ssb",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "stall_mio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    hdr = next(r)
    units = next(r)
    res = []
    for vals in r:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name", "")[:60], "id": d.get("ID", "")}
        for k, short in KEYS.items():
            if k in d:
                v = d[k].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                unit = u.get(k, "")
                if short == "dur" and unit == "usecond":
                    v = v * 1e3
                if short == "dur" and unit == "msecond":
                    v = v * 1e6
                if short.startswith("dram_") and short != "dram_pct":
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                    v = v * scale
                item[short] = v
        res.append(item)
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    rs = rows(rep)
    for it in rs:
        dur = it.get("dur", 0)
        tb = (it.get("dram_rd", 0) + it.get("dram_wr", 0))
        print(f"{it['id']:>3} {it['kernel'][:44]:44s} dur={dur/1e3:9.1f}us dram={tb/1e9:7.3f}GB "
              f"({tb/dur if dur else 0:6.0f} GB/s, {it.get('dram_pct',0):5.1f}%) regs={it.get('regs','')} "
              f"occ={it.get('occ_pct',0):5.1f}% issue={it.get('issue_pct',0):5.1f}% fp64={it.get('fp64_pct',0):5.1f}% "
              f"lsb={it.get('stall_lsb',0):.1f} bar={it.get('stall_bar',0):.1f} mio={it.get('stall_mio',0):.1f} "
              f"math={it.get('stall_math',0):.1f} l2hit={it.get('l2_hit',0):.0f}")
    if "--json" in sys.argv:
        json.dump(rs, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
