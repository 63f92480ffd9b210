# developer check: threaded host copies in the staged transfers
python -m pytest -q -x tests/test_gpu_march_api.py tests/test_gpu_parity.py -k "host or snapshot or stream or load or budget or timing" 2>&1 | tail -n 1
for i in 1 2; do python tools/e2e_phases.py double 2>&1 | grep -v Warn; done
python tools/e2e_phases.py single 2>&1 | grep -v Warn
nproc
