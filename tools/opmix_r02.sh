#!/bin/bash
# ncu source counters of the C2 fp64 theta / rho kernels (one launch each),
# aggregated by SASS opcode on the box.  Usage: bash tools/opmix_r02.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
for K in ${KERNELS:-k_rho k_theta_c2r k_theta_r2c}; do
  ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on \
      --kernel-name-base demangled -k regex:"${K}<" --launch-skip 4 -c 1 -f -o gpurun_out/${T}_src_${K} \
      python tools/rho_probe.py double "" > gpurun_out/${T}_src_${K}.log 2>&1
  echo "ncu $K rc=$?"
  ncu -i gpurun_out/${T}_src_${K}.ncu-rep --page source --csv --print-source sass \
      > gpurun_out/${T}_src_${K}.csv 2> gpurun_out/${T}_src_${K}.err
  python tools/ncu_opmix.py gpurun_out/${T}_src_${K}.csv > gpurun_out/${T}_opmix_${K}.txt 2>&1
  gzip -f gpurun_out/${T}_src_${K}.csv
  rm -f gpurun_out/${T}_src_${K}.ncu-rep
done
