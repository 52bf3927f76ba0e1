# k_mn2_scatter v2 (ranks from the counting atomic kept in registers, direct sort stores, run atomics consumed
# after the sort) at 2 blocks/SM (A, 32 regs + spill) and 1 block/SM (X1, 53 regs), vs C4 (count change only) and
# H (HEAD): multinomial / residual bit-exact tests on A, then same-box PF-step and config-5 timings
L=paper_1306_5583_b200
unset SMC_LIB_PATH
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_resample.py "tests/test_gpu_fullsize.py::test_resample_2e24_pf_weights_explicit_u_bit_exact" "tests/test_gpu_fullsize.py::test_resample_2e24_pf_weights_stream_n_bit_exact" tests/test_gpu_fullsize.py::test_multinomial_wide_bins_bit_exact tests/test_gpu_fullsize.py::test_multinomial_past_shared_memory_bins_bit_exact 2>&1 | tail -3
V="H C4 A X1"
for i in 1 2; do for v in $V; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  for sc in multinomial residual; do
    echo "$v$i $sc $(timeout 300 python bench.py --steps 40 --warmup 5 --scheme $sc --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['phase_ms']['resample'],4))")"
  done
  timeout 600 python tools/bench_resample.py --min-log2 24 --max-log2 26 --schemes multinomial,residual --kinds uniform,skewed1 --out gpurun_out/g41_mb_$v$i.jsonl > /dev/null 2>&1
  python -c "
import json
for l in open('gpurun_out/g41_mb_$v$i.jsonl'):
    d=json.loads(l); print('   $v$i mb', d.get('log2n'), d.get('scheme'), d.get('weights'), round(d.get('ms'),4))"
done; done
unset SMC_LIB_PATH
