# GMM MH blocks per SM (GMM_MIN_BLOCKS 4 shipped vs 5, 6): config-3 timing
L=paper_1306_5583_b200
for r in 1 2; do for v in cur G5 G6; do
  if [ $v = cur ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$L/libsmcb200_$v.so; fi
  timeout 300 python -c "
import bench, paper_1306_5583_b200 as P
g = bench.gmm_bench(P)
print('$v$r', round(g['ms_per_run'], 1), g['log_zconst_ds'])
" 2>&1 | tail -1
done; done
