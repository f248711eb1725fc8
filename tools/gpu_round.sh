#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, the ncu launch list of the same bench command and
# one `--set full` capture each of k_prec_coop and k_schur_explicit. Summarise afterwards (CPU side) with
#   python tools/summarize_ncu.py
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
[ -n "${TIMERS:-}" ] && timeout 300 python tools/prec_timers.py c5 > gpurun_out/timers.log 2>&1 && head -4 gpurun_out/timers.log
timeout 400 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"; tail -c 600 gpurun_out/bench.json
if [ "${1:-}" != "noncu" ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
[ "${1:-}" = "launches" ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prec_coop --launch-skip 40 -c 1 \
  -f -o gpurun_out/prec_coop python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full1.log 2>&1; echo "ncu full prec exit $?"
[ "${1:-}" = "launches" ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_schur_explicit --launch-skip 40 -c 1 \
  -f -o gpurun_out/schur_explicit python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1; echo "ncu full schur exit $?"
fi
