#!/bin/bash
# Quick GPU check: build, GPU tests, smoke, FP64 peaks, one bench line.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-}" = "" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_gpu.log
timeout 400 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
fi
[ -x tools/fp64_peak.bin ] && timeout 120 tools/fp64_peak.bin > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"; tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
