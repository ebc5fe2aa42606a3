#!/usr/bin/env python
"""NEXT-2 V2 vs D5 on the BASELINE phantoms (GPU): where the material enters the E right-hand sides.

    python tools/v2_study.py [--out gpurun_out/v2_study.json]

For c3 (64^3, p = 3, head phantom, pulse dipole, 200 steps) and c4 (128^3, p = 2, 500 steps):
  * stability: the discrete M-norm energy 1/2 (e^T M e + h^T M h) (adi_energy) every 20 steps for
    D5 (row factors of the test function, the paper-literal reading) and V2 (element material
    inside the quadrature), zero initial fields, the source driving both;
  * accuracy proxy: the relative L2 difference between the two readings per field after all steps
    (no exact solution exists for the phantom; SURVEY §8(f) asks for the empirical comparison);
  * cost: CUDA-event time of one step of each variant (the V2 E right-hand sides run as Gauss-point
    passes, everything else shared).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2103_06998_b200 as adi  # noqa: E402
import workloads  # noqa: E402


def run(cfg_name, variant, every=20):
    cfg = workloads.CONFIGS[cfg_name]
    n, p, tau, steps = cfg["n"], cfg["p"], cfg["tau"], cfg["steps"]
    N = n + p
    G = adi.Patch(n, p, tau)
    G.set_materials(workloads.element_eps(n, cfg["material"]))
    G.set_rhs_variant(variant)
    G.set_fields([np.zeros(N ** 3) for _ in range(6)])
    G.set_point_source(2, workloads.dipole_position(n), workloads.signal(cfg["source"], tau, steps))
    energy = []
    G.synchronize()
    t0 = time.perf_counter()
    for k in range(0, steps, every):
        G.step(min(every, steps - k))
        energy.append((k + min(every, steps - k), G.energy()[1]))
    G.synchronize()
    wall = time.perf_counter() - t0
    fields = G.get_fields()
    G.set_timing(True)
    G.step(2)
    G.synchronize()
    rep = G.timing_report()
    G.close()
    ms = sum(v[0] for v in rep.values()) / 2.0
    return fields, energy, ms, wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "v2_study.json"))
    ap.add_argument("--configs", default="c3,c4")
    a = ap.parse_args()
    out = {}
    for name in a.configs.split(","):
        f5, e5, ms5, w5 = run(name, 0)
        f2, e2, ms2, w2 = run(name, 2)
        diff = [float(np.linalg.norm(x - y) / max(np.linalg.norm(x), 1e-300)) for x, y in zip(f5, f2)]
        out[name] = dict(
            energy_D5=e5, energy_V2=e2, rel_diff_V2_vs_D5=diff,
            max_energy_D5=max(v for _, v in e5), max_energy_V2=max(v for _, v in e2),
            final_energy_ratio_V2_over_D5=e2[-1][1] / e5[-1][1] if e5[-1][1] else None,
            ms_per_step_D5=ms5, ms_per_step_V2=ms2, wall_s_D5=w5, wall_s_V2=w2)
        print(name, json.dumps({k: v for k, v in out[name].items() if not k.startswith("energy_")}), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
