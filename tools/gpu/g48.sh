# pass C (k_rs_assign, index-only) at 8 blocks/SM: 32 registers, store staging aliased onto the parent staging
# (25.9 KB shared instead of 35.4).  C8 = variant, H = HEAD.  Resample tests on C8, hash, same-box bench.
L=paper_1306_5583_b200
export SMC_LIB_PATH=$PWD/$L/libsmcb200_C8.so
echo "C8 tests: $(timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_resample.py tests/test_gpu_fullsize.py -k 'not mc_error and not every_step and not gmm and not strict' 2>&1 | tail -1)"
for v in H C8; do
  export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so
  echo "$v hash $(PYTHONPATH=. timeout 300 python tools/state_hash.py 1048576 8 2>&1 | tail -1)"
done
for i in 1 2 3; do for v in H C8; do
  export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so
  for sc in systematic stratified; do
  echo "$v$i $sc $(timeout 300 python bench.py --steps 60 --warmup 5 --scheme $sc --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['phase_ms']['resample'],4))")"
  done
done; done
unset SMC_LIB_PATH
