set -x
python -m pytest -q -x tests/test_gpu_parity.py -k rho_half 2>&1 | tail -2
for L in "" variants/minb6/libnwb200.so variants/minb7/libnwb200.so; do
  echo "== lib $L"
  NWB_LIB=$L python tools/rho_probe.py double "" "NWB_MAXPROD_H=8" "NWB_THETA_ROWS=1" "NWB_THETA_ROWS=1,NWB_MAXPROD_H=8" 2>&1 | grep -v Warn
done
