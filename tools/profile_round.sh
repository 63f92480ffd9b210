#!/bin/bash
# Round profiling recipe (B200_PROFILING.md), run on the GPU box from the repo root:
#   part A: plain bench (must exit 0) + clocks, then the launch list of the same
#           command with gpu__time_duration only;
#   part B/C: one `ncu --set full` capture of one full C2 step in fp64 / fp32.
# Outputs land in gpurun_out/ (scratch, <= 64 MiB per call); summaries are
# copied to profiles/.
set -x
TAG=${1:-r01b}
PART=${2:-A}
if [ "$PART" = A ]; then
  python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
  nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/${TAG}_clocks.csv
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2_f64.csv \
      python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-fp32 > gpurun_out/${TAG}_ncu_launch.log 2>&1
elif [ "$PART" = B ]; then
  timeout 900 ncu --set full --clock-control none -k regex:"k_theta|k_weno|k_rho" -s 16 -c 8 \
      -o gpurun_out/${TAG}_full_c2_f64 python tools/rho_probe.py double "" > gpurun_out/${TAG}_ncu_full64.log 2>&1
else
  timeout 900 ncu --set full --clock-control none -k regex:"k_theta|k_weno|k_rho" -s 16 -c 8 \
      -o gpurun_out/${TAG}_full_c2_f32 python tools/rho_probe.py single "" > gpurun_out/${TAG}_ncu_full32.log 2>&1
fi
ls -la gpurun_out/
