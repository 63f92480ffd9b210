"""Static SASS opcode counts per kernel of libnwb200.so (cuobjdump -sass):
evidence of the sm_100a instruction mix (TMA bulk copies UBLKCP + mbarrier
SYNCS, packed FP32 FFMA2/FADD2/FMUL2, FP64 DFMA, cp.async LDGSTS, ...).

    python tools/sass_static.py [lib] > profiles/r02_sass_static.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2103_06080_b200/libnwb200.so"
KEEP = ("DFMA", "DMUL", "DADD", "FFMA2", "FADD2", "FMUL2", "FFMA", "LDS", "STS", "LDG", "STG",
        "LDGSTS", "UBLKCP", "UBLKPF", "UTMALDG", "UTMASTG", "SYNCS", "MUFU", "BAR", "SHFL",
        "ATOMG", "REDG")

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
fams = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        fam = re.sub(r"\(.*", "", dem).replace("nwb::", "")
        cur = fams.setdefault(fam, collections.Counter())
        continue
    if cur is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
    if m:
        op = m.group(2)
        if op in KEEP:
            cur[op] += 1
print(f"static SASS opcode counts per kernel instantiation ({LIB}, cuobjdump -sass)")
for fam, c in fams.items():
    if not c:
        continue
    print(f"{fam}\n   " + "  ".join(f"{k}={c[k]}" for k in KEEP if c[k]))
