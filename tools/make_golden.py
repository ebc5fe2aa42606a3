#!/usr/bin/env python
"""Write the full-horizon oracle goldens of the north-star configs (tests/golden/<cfg>.npz).

    python tools/make_golden.py c3|c4|c5

Calls ONLY ``oracle/`` (the plain single-threaded C oracle) and ``workloads/`` (the seeded
input generators): no value here comes from the CUDA path.  The GPU test
``tests/test_golden_parity.py`` regenerates the same inputs, runs the library for the same
number of steps and compares against what this script stored.

Recipes (BASELINE.json configs; readings D9/D15 in DESIGN.md):
  c3: 64^3, p=3, phantom3 materials (D6 map of the element values), E0 = H0 = 0, Gaussian-pulse
      point dipole on E3 (D9), tau = 1e-2, 200 steps
  c4: 128^3, p=2, phantom4, E0 = H0 = 0, modulated-sine dipole on E3, tau = 1e-2, 500 steps
  c5: 512^3, p=2, phantom5, seeded random E0/H0 (workloads.random_fields(N, 55): the oracle
      cannot L2-project u_A at this size in reasonable time), no source, tau = 1e-2, 1 step
      (the oracle needs ~20 min and ~35 GB of host memory per step here)

Stored per field c (E1..H3): the full coefficient-vector norm ||x_c||_2, the sum, the max |x|,
and K sampled coefficients: K/2 seeded uniform indices plus the K/2 indices of largest |x_c|
(where a source-driven field lives), with their values.  The D16 parity metric
||x_gpu - x_orc|| / ||x_orc|| is estimated on the samples; the norms check the whole vector.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
K = 16384

RECIPES = {
    "c3": dict(steps=200, init="zero", source="pulse"),
    "c4": dict(steps=500, init="zero", source="modsine"),
    "c5": dict(steps=1, init="random", seed=55, source=None),
}


def inputs(name: str):
    """The seeded inputs of the golden run (shared with tests/test_golden_parity.py)."""
    cfg = dict(workloads.CONFIGS[name])
    rc = RECIPES[name]
    n, p, tau = cfg["n"], cfg["p"], cfg["tau"]
    N = n + p
    eps = workloads.element_eps(n, cfg["material"])
    if rc["init"] == "zero":
        fields = [np.zeros(N ** 3) for _ in range(6)]
    else:
        fields = workloads.random_fields(N, rc["seed"])
    src = None
    if rc["source"] is not None:
        src = (2, workloads.dipole_position(n), workloads.signal(rc["source"], tau, rc["steps"]))
    return dict(n=n, p=p, tau=tau, N=N, steps=rc["steps"], eps=eps, fields=fields, source=src)


def sample_indices(x: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    uni = rng.integers(0, x.size, size=K // 2)
    top = np.argpartition(np.abs(x), x.size - K // 2)[x.size - K // 2:]
    return np.unique(np.concatenate([uni, top])).astype(np.int64)


CKPT = os.path.join(ROOT, "build", "golden_ckpt")
CHUNK = 25
THREADS = int(os.environ.get("ORC_THREADS", os.cpu_count() or 1))


def _patch(I, fields, m0):
    """A fresh oracle patch holding ``fields`` after m0 steps: the source signal is shifted by m0
    (the oracle reads signal[step_index], step_index counting from 0 on a fresh patch), so resuming
    performs exactly the arithmetic of an uninterrupted run."""
    P = oracle.Patch(I["n"], I["p"], I["tau"])
    P.set_threads(THREADS)  # bit-identical to one thread (oracle header; test_threads_bit_identical)
    P.set_materials(I["eps"])
    P.set_fields(fields)
    if I["source"] is not None:
        comp, pos, sig = I["source"]
        loads = [None, None, None]
        loads[comp] = P.point_load(*pos)
        P.set_source(loads, sig[m0:])
    return P


def main(name: str):
    t0 = time.time()
    I = inputs(name)
    fields, m0, spent = I.pop("fields"), 0, 0.0
    ck = os.path.join(CKPT, f"{name}.npz")
    if os.path.exists(ck):  # resume a chunked run (checkpoints hold oracle output only)
        d = np.load(ck)
        fields, m0, spent = [d[f"f{c}"] for c in range(6)], int(d["m"]), float(d["spent"])
        print(f"{name}: resuming after {m0} steps", flush=True)
    P = _patch(I, fields, m0)
    del fields
    t1 = time.time()
    m = m0
    while m < I["steps"]:
        k = min(CHUNK, I["steps"] - m) if I["steps"] > CHUNK else I["steps"] - m
        P.step(k)
        m += k
        if m < I["steps"]:
            os.makedirs(CKPT, exist_ok=True)
            np.savez(ck + ".tmp.npz", m=m, spent=spent + time.time() - t1,
                     **{f"f{c}": x for c, x in enumerate(P.get_fields())})
            os.replace(ck + ".tmp.npz", ck)
            print(f"{name}: {m}/{I['steps']} steps, {time.time() - t1:.0f} s", flush=True)
    t2 = time.time()
    t2 += spent
    out = {"steps": I["steps"], "n": I["n"], "p": I["p"], "tau": I["tau"],
           "oracle_seconds": t2 - t1, "setup_seconds": t1 - t0}
    with open(os.path.join(ROOT, "oracle", "adi_oracle.c"), "rb") as f:
        out["oracle_sha256"] = np.frombuffer(hashlib.sha256(f.read()).digest(), dtype=np.uint8)
    fs = P.get_fields()
    norms, sums, maxs = [], [], []
    for c, x in enumerate(fs):
        idx = sample_indices(x, 1000 + c)
        out[f"idx{c}"] = idx
        out[f"val{c}"] = x[idx]
        norms.append(np.linalg.norm(x))
        sums.append(x.sum())
        maxs.append(np.abs(x).max())
    out["norm"], out["sum"], out["maxabs"] = np.array(norms), np.array(sums), np.array(maxs)
    os.makedirs(GOLD, exist_ok=True)
    path = os.path.join(GOLD, f"{name}_golden.npz")
    np.savez_compressed(path + ".tmp.npz", **out)
    os.replace(path + ".tmp.npz", path)
    if os.path.exists(ck):
        os.remove(ck)
    print(f"{name}: {I['steps']} steps in {t2 - t1:.1f} s (setup {t1 - t0:.1f} s); norms {norms}; wrote {path}",
          flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
