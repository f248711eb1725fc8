#!/bin/bash
# End-of-round measurement at HEAD: all GPU tests (per-test timeout), smoke, bench lines of c5 (default, with e2e and the
# CPU baseline), c4, c2 and c3, the ncu launch lists of the c5 and c4 bench commands and --set full captures of the top
# kernels. (compute-sanitizer is closed on this GPU pool.)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
t0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $? in $(( $(date +%s) - t0 )) s"; tail -12 gpurun_out/pytest_gpu.log
timeout 400 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 exit $?"; head -c 300 gpurun_out/bench_c5.json; echo
for cfg in c4 c2 c3; do
timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg exit $?"; head -c 200 gpurun_out/bench_$cfg.json; echo
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
for k in k_prec_coop k_schur_explicit; do
timeout 500 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 40 -c 1 -f -o gpurun_out/r2_$k \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$k.log 2>&1; echo "ncu full $k exit $?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c4.csv \
  python bench.py --config c4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu launches c4 exit $?"
for k in k_prec_coop k_schur_blk k_band_chol_panel; do
timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 -f -o gpurun_out/r2_c4_$k \
  python bench.py --config c4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c4_$k.log 2>&1; echo "ncu full c4 $k exit $?"
done
