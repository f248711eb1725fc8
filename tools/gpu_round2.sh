#!/bin/bash
# Round-2 measurement call: all GPU tests, smoke, FP64 peaks, default bench line (c5) and a c4 line, the ncu launch
# list of the bench command, --set full captures of the top kernels (c5 and c4), compute-sanitizer runs.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -22 gpurun_out/pytest_gpu.log
timeout 400 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
fi
timeout 120 tools/fp64_peak.bin > gpurun_out/fp64_peak.json 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 exit $?"; head -c 400 gpurun_out/bench_c5.json; echo
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 exit $?"; head -c 400 gpurun_out/bench_c4.json; echo
if [ -z "${SKIP_NCU:-}" ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
for k in k_prec_coop k_schur_explicit; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 40 -c 1 -f -o gpurun_out/r2_$k \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$k.log 2>&1; echo "ncu full $k exit $?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c4.csv \
  python bench.py --config c4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu launches c4 exit $?"
for k in k_prec_coop k_schur_blk k_band_chol_panel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 -f -o gpurun_out/r2_c4_$k \
  python bench.py --config c4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c4_$k.log 2>&1; echo "ncu full c4 $k exit $?"
done
fi
if [ -z "${SKIP_SAN:-}" ]; then
timeout 1200 compute-sanitizer --tool memcheck --leak-check none python tools/sanitize_run.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck exit $?"; tail -3 gpurun_out/sanitize_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_run.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck exit $?"; tail -3 gpurun_out/sanitize_racecheck.log
fi
