python -c "from paper_1306_5583_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_resample.py tests/test_gpu_dist.py tests/test_gpu_dist_sampler.py tests/test_gpu_edges.py -x -q -p no:randomly > gpurun_out/pytest_mn.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_mn.log
for v in A OLD; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/paper_1306_5583_b200/libsmcb200_OLD.so; fi
  echo "== $v"; timeout 600 python tools/bench_resample.py --min-log2 20 --max-log2 24 --step 2 --schemes multinomial,residual,systematic --kinds uniform,skewed1,degenerate 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d.get('scheme'), d.get('weights', d.get('kind')), d.get('log2n', d.get('n')), round(d.get('ms',0),4))
"
done
unset SMC_LIB_PATH
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_mn2.csv python tools/prof_multinomial.py > /dev/null 2>&1; echo ncu rc=$?
timeout 900 python -m pytest tests/test_gpu_gmm.py -x -q -p no:randomly > gpurun_out/pytest_gmm.log 2>&1; echo "pytest gmm rc=$?"; tail -3 gpurun_out/pytest_gmm.log
bash tools/ab_lib.sh "python tools/bench_gmm.py --seeds 1 2>/dev/null | tail -1 | cut -c1-200" A OLD
