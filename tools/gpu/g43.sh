# (second run: the count kernel loads the floors with Q) residual-multinomial: pass A seeds the draws' histogram with the floors f_i, the count kernel adds onto them and
# pass B1 reads the finished counts (no second quantization from the log-weights).  A = new, H = HEAD.
L=paper_1306_5583_b200
unset SMC_LIB_PATH
timeout 1800 python -m pytest -q -x -m gpu tests/test_gpu_resample.py tests/test_gpu_fullsize.py -k "not mc_error and not every_step and not gmm and not strict" tests/test_gpu_dist_sampler.py tests/test_gpu_dist.py tests/test_gpu_bench_multirank.py 2>&1 | tail -3
timeout 900 python -m pytest -q -x -m gpu "tests/test_gpu_fullsize.py::test_pf_2e24_100_obs_resampling_bit_exact_every_step[residual]" "tests/test_gpu_fullsize.py::test_pf_2e24_100_obs_resampling_bit_exact_every_step[multinomial]" 2>&1 | tail -2
for i in 1 2; do for v in H A; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  for sc in residual multinomial; do
    echo "$v$i $sc $(timeout 300 python bench.py --steps 40 --warmup 5 --scheme $sc --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['phase_ms']['resample'],4))")"
  done
  timeout 600 python tools/bench_resample.py --min-log2 24 --max-log2 26 --schemes multinomial,residual --kinds uniform,skewed1,degenerate --out gpurun_out/g43_mb_$v$i.jsonl > /dev/null 2>&1
  python -c "
import json
for l in open('gpurun_out/g43_mb_$v$i.jsonl'):
    d=json.loads(l); print('   $v$i mb', d.get('log2n'), d.get('scheme'), d.get('weights'), round(d.get('ms'),4))"
done; done
unset SMC_LIB_PATH
