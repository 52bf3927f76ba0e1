# GMM likelihood with the (y, y^2) quadratic expansion: GMM GPU tests (incl. config 3 at full size vs the
# oracle) on the new library, then same-box config-3 timing A (new, 4 blocks/SM) / G0 (HEAD) / G5 (new, 5/SM)
L=paper_1306_5583_b200
unset SMC_LIB_PATH
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_gmm.py "tests/test_gpu_fullsize.py::test_gmm_config3_first_iterations_match_oracle" 2>&1 | tail -3
for i in 1 2; do for v in A G0 G5; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  echo "$v$i $(timeout 300 python tools/bench_gmm.py --seeds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['runs'][0]; print(round(d['ms_per_run'],1), r['log_z_ds'], r['log_z_ps'], r['acc_rate_mu'])")"
done; done
unset SMC_LIB_PATH
