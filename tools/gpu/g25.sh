# ncu --set full of k_rs_assign<0,1> and k_rs_tiles (W input), stratified uniform 2^24: round-1 library vs current
for v in r1 cur; do
  if [ $v = r1 ]; then export SMC_LIB_PATH=tools/gpu/r1/libsmcb200.so; else unset SMC_LIB_PATH; fi
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rs_assign|k_rs_tiles" -s 4 -c 2 -o gpurun_out/g25_$v python tools/bench_resample.py --min-log2 24 --max-log2 24 --schemes stratified --kinds uniform > gpurun_out/g25_$v.log 2>&1; echo "$v rc=$?"
done
