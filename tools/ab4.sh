python -m paper_1501_06211_b200.build > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "precond or lanczos" 2>&1 | tail -1
for v in 0 1; do
  if [ $v = 1 ]; then cp _ab/libde_base.so paper_1501_06211_b200/libde.so; fi
  echo "== arm $v"
  python tools/prec_timers.py c4 2>&1 | grep -E "precond ms|phases" | tail -2
  python tools/inner_modes.py c4 2>&1 | grep "| X"
done
