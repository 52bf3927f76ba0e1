# per-kernel durations of one stratified resample (uniform W, 2^24): round-1 library vs current
for v in r1 cur; do
  if [ $v = r1 ]; then export SMC_LIB_PATH=tools/gpu/r1/libsmcb200.so; else unset SMC_LIB_PATH; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rs_ -c 60 --csv --log-file gpurun_out/g24_$v.csv python tools/bench_resample.py --min-log2 24 --max-log2 24 --schemes stratified,systematic --kinds uniform > /dev/null 2>&1; echo "$v rc=$?"
done
