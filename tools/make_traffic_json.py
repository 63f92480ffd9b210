"""Write profiles/ncu_traffic.json from an `ncu --set full` report.

    python tools/make_traffic_json.py REPORT.ncu-rep CONFIG PRECISION

Per kernel group (theta_c2r, weno, theta_r2c, rho_pass) the average
dram__bytes_read.sum + dram__bytes_write.sum per launch; bench.py reports it
as roofline.traffic beside the algorithmic bytes.
"""

import csv
import json
import os
import subprocess
import sys

GROUPS = {"k_theta_c2r": "theta_c2r", "k_theta_r2c": "theta_r2c", "k_weno": "weno", "k_weno_x2": "weno",
          "k_rho": "rho_pass", "k_rho_r80": "rho_pass"}


def scale(v, unit):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(rep, config, precision):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    it = hdr.index("gpu__time_duration.sum")
    pipes = {k: hdr.index(m) for k, m in (
        ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        ("issue_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed")) if m in hdr}
    acc = {}
    for d in data:
        name = d[hdr.index("Kernel Name")].split("<")[0].replace("void ", "").split("::")[-1]
        g = GROUPS.get(name)
        if not g:
            continue
        b = scale(d[ir], units[ir]) + scale(d[iw], units[iw])
        e = acc.setdefault(g, {"bytes": 0.0, "n": 0, "us": 0.0, **{k: 0.0 for k in pipes}})
        for k, i in pipes.items():
            e[k] += float(d[i])
        e["bytes"] += b
        e["n"] += 1
        e["us"] += float(d[it]) * (1e-3 if units[it] == "ns" else 1.0)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "ncu_traffic.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    table.setdefault(config, {})[precision] = {
        g: {"dram_bytes_per_launch": round(e["bytes"] / e["n"]), "launches": e["n"],
            "ncu_us_per_launch": round(e["us"] / e["n"], 1), "report": os.path.basename(rep),
            **{k: round(e[k] / e["n"], 1) for k in pipes}}
        for g, e in acc.items()}
    with open(path, "w") as fh:
        json.dump(table, fh, indent=1, sort_keys=True)
    print(json.dumps(table[config][precision], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
