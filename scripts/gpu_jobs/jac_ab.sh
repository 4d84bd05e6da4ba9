# A/B of the Jacobian kernel builds present in _lib (default first), then the Jacobian parity tests
for L in "" $(ls paper_1409_2556_b200/_lib/liblaptomo_gpu_*.so 2>/dev/null); do
  if [ -z "$L" ]; then unset LT_LIB; else export LT_LIB=$PWD/$L; fi
  timeout 600 python scripts/jac_ab.py 2>&1 | tail -1
done
unset LT_LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_split.py -q -x 2>&1 | tail -3
