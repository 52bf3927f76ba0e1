# k_mn2_scatter draws per thread (occupancy) A/B: PF multinomial / residual + microbench multinomial
L=paper_1306_5583_b200
for r in 1 2; do for v in cur CA CB; do
  if [ $v = cur ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$L/libsmcb200_$v.so; fi
  for sc in multinomial residual; do
    timeout 600 python bench.py --scheme $sc --steps 30 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e --no-config1 --no-schemes > gpurun_out/g30_$v$sc$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/g30_$v$sc$r.json').read().strip().splitlines()[-1]);print('$v $sc $r',round(d['ms_per_step'],4),d['phase_ms'])"
  done
  timeout 600 python tools/bench_resample.py --min-log2 24 --max-log2 26 --schemes multinomial,residual --kinds uniform,skewed1 --out gpurun_out/g30_$v$r.jsonl > /dev/null 2>&1
done; done
unset SMC_LIB_PATH
python tools/ab_resample_table.py gpurun_out/g30 cur CA CB
