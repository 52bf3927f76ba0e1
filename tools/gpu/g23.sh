# resample microbench A/B (r1 lib, r2 before today, current, current + philox10 draw53) + multinomial tests
L=paper_1306_5583_b200
timeout 1500 python -m pytest tests/test_gpu_resample.py tests/test_gpu_fullsize.py -k "multinomial or residual or past_shared or explicit" -m gpu -q -p no:randomly > gpurun_out/g23_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g23_pytest.log
for r in 1 2; do for v in r1 old cur S; do
  case $v in r1) export SMC_LIB_PATH=tools/gpu/r1/libsmcb200.so;; old) export SMC_LIB_PATH=tools/gpu/old/libsmcb200.so;; cur) unset SMC_LIB_PATH;; S) export SMC_LIB_PATH=$L/libsmcb200_S.so;; esac
  timeout 600 python tools/bench_resample.py --min-log2 24 --max-log2 26 --schemes systematic,stratified,multinomial,residual,residual_stratified,residual_systematic --kinds uniform,skewed1,degenerate --out gpurun_out/g23_$v$r.jsonl > /dev/null 2>&1; echo "$v$r rc=$?"
done; done
unset SMC_LIB_PATH
