#!/bin/bash
# Developer tool: A/B of library variants on the C2 fp64 bench (device-resident):
#   tools/ab_bench.sh <rounds> <lib1> <lib2> ...   (NWB_LIB selects the library)
R=$1; shift
for i in $(seq $R); do
  for L in "$@"; do
    NWB_LIB=$L python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-fp32 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$L', round(d['ms_per_step'],4), [(k['kernel'],round(k['ms'],4)) for k in d['roofline']['per_kernel'][:4]])"
  done
done
