#!/bin/bash
# A/B of environment switches on the GPU box: AB_VARIANTS="|DE_NO_PAT=1|DE_NO_SPLIT=1 DE_NO_PAT=1" (| separated; the
# empty variant is the default build), AB_CONFIGS="c5 c4", AB_TESTS = pytest -k expression (default: the
# preconditioner parity tests), AB_BENCH=1 adds a short bench line per variant.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gram_cgs2.py tests/test_cross_fd.py -m gpu -q -x -k "${AB_TESTS:-precond or lanczos or gram or fd}" 2>&1 | tail -3
IFS='|' read -ra VARS <<< "${AB_VARIANTS:-|DE_NO_PAT=1}"
for cfg in ${AB_CONFIGS:-c5}; do
for envs in "${VARS[@]}"; do
  echo "== $cfg [$envs]"
  env $envs timeout 300 python tools/prec_ab.py $cfg 30 2>&1 | tail -1
  env $envs DE_PREC_TIMERS=1 timeout 300 python tools/prec_ab.py $cfg 10 2>&1 | tail -2
  if [ -n "${AB_BENCH:-}" ]; then
    env $envs timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BENCH', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'its', d['iterations_per_step'], 'factor', round(d['factor_ms'],2), 'prec', round(d['roofline']['launch_ms'],4), 'schur', round(d['roofline_secondary']['launch_ms'],4))"
  fi
done
done
