"""Full-length BASELINE C2 parity ("optionally one cached
full-length golden"): the whole 2400-step Set-4 march of the bench's input
(rho-modulated N-wave, fp64) on the B200 through run_exprk22, against the CPU
oracle (the reference's arithmetic, bitwise-pinned to reference goldens) on
the box's host cores.  Writes gpurun_out/full_c2_parity.json."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_06080_b200 as nw  # noqa: E402
from oracle import nwave_oracle as oracle  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "double"
c2 = nw.preset_config(4)
_, rho, theta = nw.build_axes(c2)
v0 = nw.rho_modulated(c2, nw.initial_nwave(rho, theta, c2.A, c2.B))
f = nw.zero_fields(c2.N_sigma + 1, c2.N_rho + 1)
t0 = time.perf_counter()
rep = nw.run_exprk22(c2, v0, f, precision=prec, snapshot_sigmas=[30.0, 60.0, 90.0])
t_gpu = time.perf_counter() - t0
t0 = time.perf_counter()
ref = oracle.march(c2, v0.values, f, precision=prec, snapshot_sigmas=[30.0, 60.0, 90.0])
t_cpu = time.perf_counter() - t0
a, b = ref.final, rep.final.values
res = {
    "config": "C2 Set 4 10000x3584, rho-modulated N-wave, full N_sigma = 2400 steps",
    "precision": prec,
    "max_relative_final": float(np.max(np.abs(a - b)) / np.max(np.abs(a))),
    "rel_l2_final": float(np.linalg.norm(a - b) / np.linalg.norm(a)),
    "max_relative_snapshots": {str(s): float(np.max(np.abs(ref.snapshots[s] - rep.snapshots[s].values))
                                             / np.max(np.abs(ref.snapshots[s])))
                               for s in (30.0, 60.0, 90.0)},
    "max_abs_v_gpu": rep.max_abs_v, "max_abs_v_oracle": ref.max_abs_v,
    "gpu_run_s": t_gpu, "cpu_oracle_s": t_cpu, "cpu_cores": oracle.host_cores(),
}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"full_c2_parity_{prec}.json"), "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res))
