# residual-stratified / -systematic: pass B1 reads q'_i (pass A's qfull) and f_i (pass A, the histogram buffer)
# instead of re-quantizing from the log-weights.  A = new, H = HEAD.
L=paper_1306_5583_b200
unset SMC_LIB_PATH
timeout 1800 python -m pytest -q -x -m gpu tests/test_gpu_resample.py tests/test_gpu_fullsize.py -k "not mc_error and not every_step and not gmm and not strict" tests/test_gpu_dist_sampler.py tests/test_gpu_dist.py tests/test_gpu_bench_multirank.py tests/test_gpu_weights_pf.py 2>&1 | tail -3
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fullsize.py -k "every_step" 2>&1 | tail -2
for i in 1 2; do for v in H A; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  for sc in residual_systematic residual_stratified residual systematic; do
    echo "$v$i $sc $(timeout 300 python bench.py --steps 40 --warmup 5 --scheme $sc --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['phase_ms']['resample'],4))")"
  done
  timeout 600 python tools/bench_resample.py --min-log2 24 --max-log2 26 --schemes residual_systematic,residual_stratified --kinds uniform,skewed1,degenerate --out gpurun_out/g44_mb_$v$i.jsonl > /dev/null 2>&1
  python -c "
import json
for l in open('gpurun_out/g44_mb_$v$i.jsonl'):
    d=json.loads(l); print('   $v$i mb', d.get('log2n'), d.get('scheme'), d.get('weights'), round(d.get('ms'),4))"
done; done
unset SMC_LIB_PATH
