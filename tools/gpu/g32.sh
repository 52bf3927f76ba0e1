# GMM likelihood exp with the 256-entry table (degree-4): GMM tests + config-3 timing A/B against HEAD
timeout 1200 python -m pytest tests/test_gpu_gmm.py tests/test_gpu_fullsize.py -k "gmm" -m gpu -q -p no:randomly > gpurun_out/g32_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g32_pytest.log
for r in 1 2; do for v in head cur; do
  if [ $v = head ]; then export SMC_LIB_PATH=tools/gpu/head/libsmcb200.so; else unset SMC_LIB_PATH; fi
  timeout 300 python -c "
import bench, paper_1306_5583_b200 as P
g = bench.gmm_bench(P)
print('$v$r', round(g['ms_per_run'], 1), g['log_zconst_ds'], g['log_zconst_ps'])
" 2>&1 | tail -1
done; done
