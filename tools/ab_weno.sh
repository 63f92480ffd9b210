#!/bin/bash
# Developer tool: WENO per-launch times of library variants at C2 (fp64 / fp32,
# tools/rho_probe.py) and C4 (bench.py --config c4): tools/ab_weno.sh lib...
for L in "$@"; do
  a=$(NWB_LIB=$L python tools/rho_probe.py double "" 2>&1 | grep -o "^double.*" | python -c "import sys,ast; l=sys.stdin.read(); v=ast.literal_eval(l[l.index(':')+1:l.index('rho sum')].strip()); print(v[1])")
  b=$(NWB_LIB=$L python tools/rho_probe.py single "" 2>&1 | grep -o "^single.*" | python -c "import sys,ast; l=sys.stdin.read(); v=ast.literal_eval(l[l.index(':')+1:l.index('rho sum')].strip()); print(v[1])")
  c=$(NWB_LIB=$L python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['roofline']['per_kernel'][1]['ms'], d['fp32']['roofline']['per_kernel'][1]['ms'])")
  echo "$L C2 f64 $a f32 $b | C4 f64/f32 $c"
done
