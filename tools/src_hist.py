"""Developer diagnostic: executed instructions / stall samples per CUDA source
line from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname, out, hdr = None, [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and r[2] == "-":
        ie, st = int(r[7] or 0), int(r[4] or 0)
        if ie or st:
            out.append((ie, st, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
tots = sum(o[1] for o in out) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for o in sorted(out, reverse=True)[:n]:
    print(f"{o[0] / tot:6.3f} stall {o[1] / tots:6.3f} {o[2]:18s} {o[3]}")
