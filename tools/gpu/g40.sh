# k_mn2_count F(X): sub-bucket scan predicated (MN_FU 4 = A, 6 = F6) vs HEAD (H): multinomial / residual bit-exact
# tests on A, then same-box PF-step and config-5 timings
L=paper_1306_5583_b200
unset SMC_LIB_PATH
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_resample.py "tests/test_gpu_fullsize.py::test_resample_2e24_pf_weights_explicit_u_bit_exact" "tests/test_gpu_fullsize.py::test_resample_2e24_pf_weights_stream_n_bit_exact" tests/test_gpu_fullsize.py::test_multinomial_wide_bins_bit_exact 2>&1 | tail -3
for v in H A F6; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  echo "$v hash $(PYTHONPATH=. timeout 300 python tools/state_hash.py 1048576 8 2>&1 | tail -1)"
done
for i in 1 2; do for v in H A F6; do
  if [ $v = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/$L/libsmcb200_$v.so; fi
  for sc in multinomial residual; do
    echo "$v$i $sc $(timeout 300 python bench.py --steps 40 --warmup 5 --scheme $sc --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['phase_ms']['resample'],4))")"
  done
  timeout 600 python tools/bench_resample.py --min-log2 24 --max-log2 24 --schemes multinomial,residual --kinds uniform,skewed1 --out gpurun_out/g40_mb_$v$i.jsonl > /dev/null 2>&1
  python -c "
import json
for l in open('gpurun_out/g40_mb_$v$i.jsonl'):
    d=json.loads(l); print('   $v$i mb', d.get('scheme'), d.get('weights'), d.get('ms'))"
done; done
unset SMC_LIB_PATH
