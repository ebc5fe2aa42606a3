"""Print key per-launch metrics from an `ncu --page raw --csv` export.

    python tools/ncu_raw.py gpurun_out/raw_c5_x.csv
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "rdGB"), ("dram__bytes_write.sum", "wrGB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"), ("lts__t_sector_hit_rate.pct", "l2hit"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "lsb"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "wait"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "ssb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "bar"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "lgthr"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "mio"),
    ("smsp__inst_executed.sum", "Ginst"), ("launch__grid_size", "grid"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    print("kernel".ljust(44) + "".join(f"{n:>8s}" for _, n in KEYS))
    for r in data:
        name = r[ix["Kernel Name"]][:43]
        vals = []
        for k, n in KEYS:
            v = r[ix[k]] if k in ix else ""
            try:
                x = float(v.replace(",", ""))
                u = units[ix[k]]
                if n == "ms":
                    x = x / 1e6 if u == "ns" else x / 1e3 if u == "us" else x
                if n in ("rdGB", "wrGB"):
                    x = x / {"byte": 1e9, "Kbyte": 1e6, "Mbyte": 1e3, "Gbyte": 1.0}.get(u, 1e9)
                if n == "Ginst":
                    x /= 1e9
                vals.append(f"{x:8.3f}" if abs(x) < 1000 else f"{x:8.0f}")
            except ValueError:
                vals.append(f"{v[:7]:>8s}")
        print(name.ljust(44) + "".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
