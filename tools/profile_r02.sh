#!/bin/bash
# Round-2 evidence run on one B200 (from the repo root): GPU tests, smoke,
# default bench + other configs, studies / splitting timings, the launch list
# and one `ncu --set full` capture of a C2 step in fp64 and fp32 (each ncu run
# only after the same command exited 0 without ncu).
T=${1:-r02a}
O=gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${T}_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${T}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/${T}_smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $O/${T}_clocks.csv &
CP=$!
python bench.py > $O/${T}_bench_c2_default.jsonl 2> $O/${T}_bench_c2.err; echo "bench rc=$?"
kill $CP
python bench.py --config c4 --steps 20 --warmup 3 --no-cpu > $O/${T}_bench_c4.jsonl 2>/dev/null; echo "c4 rc=$?"
python bench.py --config c3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/${T}_bench_c3.jsonl 2>/dev/null; echo "c3 rc=$?"
python bench.py --config c1 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/${T}_bench_c1.jsonl 2>/dev/null; echo "c1 rc=$?"
python bench.py --config c5 --steps 10 --warmup 3 > $O/${T}_bench_c5.jsonl 2>/dev/null; echo "c5 rc=$?"
python tools/study_timing.py > $O/${T}_studies.txt 2>&1; echo "studies rc=$?"
python tools/split_timing.py > $O/${T}_splitting.txt 2>&1; echo "splitting rc=$?"
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-fp32 > $O/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches_c2_f64.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-fp32 > $O/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
for p in double single; do
  python tools/rho_probe.py $p "" > $O/${T}_probe_$p.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_theta|k_weno|k_rho" -s 16 -c 8 \
      -o $O/${T}_full_c2_$p python tools/rho_probe.py $p "" > $O/${T}_ncu_full_$p.log 2>&1; echo "ncu $p rc=$?"
done
# summaries on the box (the reports are large): per-kernel table, traffic json, stalls
for p in double single; do
  python tools/ncu_summary.py $O/${T}_full_c2_$p.ncu-rep > $O/${T}_ncu_full_c2_$p.txt 2>&1
  ncu -i $O/${T}_full_c2_$p.ncu-rep --page raw --csv > $O/${T}_raw_$p.csv 2>/dev/null
done
python tools/make_traffic_json.py $O/${T}_full_c2_double.ncu-rep c2 double > $O/${T}_traffic64.log 2>&1
python tools/make_traffic_json.py $O/${T}_full_c2_single.ncu-rep c2 single > $O/${T}_traffic32.log 2>&1
cp profiles/ncu_traffic.json $O/${T}_ncu_traffic.json
gzip -f $O/${T}_raw_double.csv $O/${T}_raw_single.csv
rm -f $O/${T}_full_c2_single.ncu-rep   # keep one report under gpurun's 64 MiB return limit
ls -la $O | tail -40
