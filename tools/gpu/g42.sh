# plain move at 7 / 6 blocks per SM (M7, M6) and 2 particles interleaved at 6 (U2): hash + same-box bench
L=paper_1306_5583_b200
V="A M7 M6 U2"
for v in $V; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  echo "$v hash $(PYTHONPATH=. timeout 300 python tools/state_hash.py 1048576 8 2>&1 | tail -1)"
done
for i in 1 2; do for v in $V; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e --no-schemes --no-config1 > gpurun_out/g42_$v$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/g42_$v$i.json').read().strip().splitlines()[-1]);print('$v$i',round(d['ms_per_step'],4),d['phase_ms'])"
done; done
unset SMC_LIB_PATH
