# developer A/B: WENO tile staging by cp.async
for L in variants/base/libnwb200.so ""; do
  echo "== lib ${L:-default}"
  for p in double single; do
    NWB_LIB=$L python tools/rho_probe.py $p "" 2>&1 | grep -v Warn
    NWB_LIB=$L python tools/step_probe.py $p "" 2>&1 | grep -v Warn
  done
done
python -m pytest -q -x tests/test_gpu_parity.py 2>&1 | tail -n 1
python -m pytest -q -x tests/test_gpu_bench_configs.py -k c2 2>&1 | tail -n 1
python -m pytest -q -x tests/test_gpu_slab.py tests/test_gpu_reference_ports.py 2>&1 | tail -n 1
