# GMM likelihood loop unrolled over data points (GMM_UNROLL 2 / 4, same arithmetic order): GMM tests on each,
# then same-box config-3 timing vs H (HEAD)
L=paper_1306_5583_b200
for v in U2 U4; do
  export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so
  echo "$v tests: $(timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_gmm.py 'tests/test_gpu_fullsize.py::test_gmm_config3_first_iterations_match_oracle' 2>&1 | tail -1)"
done
for i in 1 2; do for v in H U2 U4; do
  export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so
  echo "$v$i $(timeout 300 python tools/bench_gmm.py --seeds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['runs'][0]; print(round(d['ms_per_run'],1), r['log_z_ds'], r['log_z_ps'], r['acc_rate_mu'])")"
done; done
unset SMC_LIB_PATH
