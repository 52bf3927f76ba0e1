# move variants (XU-pipe conversions replaced): bit-identity hash + same-box interleaved bench
L=paper_1306_5583_b200
for v in A H I J K; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  echo "$v hash $(PYTHONPATH=. timeout 300 python tools/state_hash.py 1048576 8 2>&1 | tail -1)"
done
for i in 1 2; do for v in A H I J K; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e --no-schemes > gpurun_out/g19_$v$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/g19_$v$i.json').read().strip().splitlines()[-1]);print('$v$i',round(d['ms_per_step'],4),d['phase_ms'])"
done; done
unset SMC_LIB_PATH
