# developer check after the fp32 rho launch-bound change
python tools/rho_probe.py single "" 2>&1 | grep -v Warn
python tools/step_probe.py single "" 2>&1 | grep -v Warn
python -m pytest -q -x tests/test_gpu_bench_configs.py -k "fp32" 2>&1 | tail -2
python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_slab.py 2>&1 | tail -2
python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; [print('c4', l.get('ms_per_step'), l.get('fp32', {}).get('ms_per_step') if isinstance(l.get('fp32'), dict) else l.get('fp32')) for l in map(json.loads, sys.stdin)]"
