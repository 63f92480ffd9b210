"""Aggregate an ncu source-page CSV (``ncu -i rep --page source --csv
--print-source sass``) by SASS opcode: executed warp instructions and stall
samples per opcode family, per kernel section.

    python tools/ncu_opmix.py source.csv > summary.txt
"""
import collections
import csv
import io
import re
import sys


def sections(text):
    """ncu prints one CSV table per profiled kernel, each preceded by a
    'Kernel Name' style line or a repeated header: split on header lines."""
    lines = text.splitlines()
    cur, head = [], None
    for ln in lines:
        if ln.startswith('"#"') or ln.startswith('"Address"') or ln.startswith("# ") or (
                ln.startswith('"') and "Source" in ln and "Address" in ln):
            if cur:
                yield head, cur
            head, cur = ln, []
        elif head is not None:
            cur.append(ln)
        else:
            print("preamble:", ln[:200])
    if cur:
        yield head, cur


def main(path):
    text = open(path, errors="replace").read()
    for head, body in sections(text):
        rows = list(csv.reader(io.StringIO("\n".join([head] + body))))
        hdr = rows[0]
        src = next((i for i, h in enumerate(hdr) if h.strip() == "Source"), None)
        exe = next((i for i, h in enumerate(hdr) if "Instructions Executed" in h and "Predicated" not in h), None)
        smp = next((i for i, h in enumerate(hdr) if "Sampling (All" in h), None)
        if src is None or exe is None:
            print("columns:", hdr)
            continue
        ops = collections.Counter()
        stalls = collections.Counter()
        tot = 0
        for r in rows[1:]:
            if len(r) <= max(src, exe):
                continue
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[src])
            if not m:
                continue
            op = m.group(2)
            try:
                n = float(r[exe] or 0)
            except ValueError:
                continue
            ops[op] += n
            tot += n
            if smp is not None:
                try:
                    stalls[op] += float(r[smp] or 0)
                except ValueError:
                    pass
        st = sum(stalls.values()) or 1
        print(f"== section ({len(rows) - 1} SASS lines), executed warp instructions {tot:.4g}")
        for op, n in ops.most_common(40):
            print(f"  {op:10s} {n:12.4g} {100 * n / tot:6.2f} %   stall samples {100 * stalls[op] / st:6.2f} %")


if __name__ == "__main__":
    main(sys.argv[1])
