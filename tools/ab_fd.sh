#!/bin/bash
# A/B of the round-2 preconditioner changes on the GPU box: fast-diagonalised cross-point solve (DE_NO_FD = dense
# S_C^-1 stream) and the split-phase arrival between t_C and the cross-point solve (DE_NO_SPLIT = grid barrier).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_cross_fd.py tests/test_gpu_parity.py tests/test_gram_cgs2.py -m gpu -q -x 2>&1 | tail -3
for cfg in "${AB_CONFIGS:-c5}"; do
for envs in "" "DE_NO_FD=1" "DE_NO_SPLIT=1" "DE_NO_FD=1 DE_NO_SPLIT=1"; do
  echo "== $cfg [$envs]"
  env $envs timeout 300 python tools/prec_ab.py $cfg 30 2>&1 | tail -1
  env $envs DE_PREC_TIMERS=1 timeout 300 python tools/prec_ab.py $cfg 10 2>&1 | tail -3
done
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err; echo "bench exit $?"; head -c 600 gpurun_out/bench_ab.json; echo
