# launch lists of the PF step under residual and multinomial (current vs round-1 library)
for v in cur r1; do
  if [ $v = r1 ]; then export SMC_LIB_PATH=tools/gpu/r1/libsmcb200.so; else unset SMC_LIB_PATH; fi
  for sc in residual multinomial; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/g27_${v}_$sc.csv python bench.py --scheme $sc --steps 5 --warmup 3 --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 > gpurun_out/g27_${v}_$sc.log 2>&1; echo "$v $sc rc=$?"
  done
done
