python -c "from paper_1306_5583_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_resample.py tests/test_gpu_dist.py tests/test_gpu_dist_sampler.py tests/test_gpu_fullsize.py -k "not 100_obs and not gmm_config3" -x -q -p no:randomly > gpurun_out/pytest_mn.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_mn.log
timeout 600 python tools/bench_resample.py --min-log2 24 --max-log2 24 --schemes multinomial,residual,systematic --kinds uniform,skewed1,degenerate 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d.get('scheme'), d.get('weights'), d.get('log2n'), round(d.get('ms',0),4))
"
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_mn2 -c 10 --csv --log-file gpurun_out/launches_mn2.csv python tools/prof_multinomial.py > /dev/null 2>&1; echo ncu rc=$?
for f in 0.3 0.55 0.7; do timeout 120 tools/tma_copy_ab 24 $f; done
timeout 120 tools/tma_copy_ab 26 0.55
