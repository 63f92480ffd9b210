"""Developer diagnostic: histogram of executed SASS instructions and stall
samples per opcode from `ncu -i X --page source --csv --print-source sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
by, stall = collections.Counter(), collections.Counter()
hdr = None
tot = tots = 0
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    op = r[1].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    n, s = int(r[ie] or 0), int(r[st] or 0)
    by[o] += n
    stall[o] += s
    tot += n
    tots += s
print("total warp inst", tot, "stall samples", tots)
for o, n in by.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{o:10s} {n:12d} {n / tot:6.3f}  stall {stall[o] / max(tots, 1):6.3f}")
