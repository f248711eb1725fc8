# A/B timing on the GPU box (tuning only): arm 0 = the working tree's libde.so, arm 1 = _ab/libde_base.so
# (or, when ABVAR is set, the same library with that environment variable set).
python -m paper_1501_06211_b200.build > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${ABTESTS:-precond or lanczos}" 2>&1 | tail -1
for v in 0 1; do
  if [ $v = 1 ]; then
    if [ -n "$ABVAR" ]; then export $ABVAR=1; else cp _ab/libde_base.so paper_1501_06211_b200/libde.so; fi
  fi
  echo "== arm $v ${ABVAR}"
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BENCH', round(d['value'],1), round(d['ms_per_step'],1), d['iterations_per_step'], 'factor', round(d['factor_ms'],2), round(d['roofline']['launch_ms'],4), round(d['roofline_secondary']['launch_ms'],4))"
done
