#!/bin/bash
for m in 1 2 4; do
ADI_SW_TMA=$m timeout 300 python - <<'PY'
import os, numpy as np, sys
sys.path.insert(0, '.')
import oracle, workloads, paper_2103_06998_b200 as adi
m = os.environ['ADI_SW_TMA']
for n, p in [(34, 2), (29, 3), (8, 2)]:
    try:
        O, G = oracle.Patch(n, p, 0.01), adi.Patch(n, p, 0.01)
        eps = workloads.element_eps(n, 'phantom4'); f = workloads.random_fields(n + p, 1)
        for X in (O, G): X.set_materials(eps); X.set_fields(f); X.step(2)
        e = max(np.linalg.norm(a - b) / np.linalg.norm(b) for a, b in zip(G.get_fields(), O.get_fields()))
        print(f"mask {m} n={n} p={p}: max rel err {e:.3e}", flush=True)
    except Exception as ex:
        print(f"mask {m} n={n} p={p}: FAILED {ex}", flush=True); break
PY
done
