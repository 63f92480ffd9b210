# developer check: kernel time stamps for the default-path buckets
python -m pytest -q -x tests/test_gpu_march_api.py tests/test_gpu_parity.py tests/test_gpu_splitting.py tests/test_gpu_slab.py 2>&1 | tail -n 2
python tools/e2e_phases.py double 2>&1 | grep -v Warn
python tools/e2e_phases.py single 2>&1 | grep -v Warn
python tools/_timing_overhead.py 2>&1 | grep -v Warn
python tools/step_probe.py double "" 2>&1 | grep -v Warn
