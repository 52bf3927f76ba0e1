# k_mn2_count particle loop with 4 steps' loads in flight: multinomial/residual tests + PF scheme sweep A/B vs HEAD
timeout 1500 python -m pytest tests/test_gpu_resample.py tests/test_gpu_fullsize.py -k "multinomial or residual or past_shared or explicit or stream" -m gpu -q -p no:randomly > gpurun_out/g28_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g28_pytest.log
for r in 1 2; do for v in head cur; do
  if [ $v = head ]; then export SMC_LIB_PATH=tools/gpu/head/libsmcb200.so; else unset SMC_LIB_PATH; fi
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e --no-config1 > gpurun_out/g28_$v$r.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/g28_$v$r.json').read().strip().splitlines()[-1]);print('$v$r',round(d['ms_per_step'],4),{k:round(x['ms_per_step'],4) for k,x in d['schemes'].items()})"
done; done
unset SMC_LIB_PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mn2 -c 40 --csv --log-file gpurun_out/g28_mn.csv python bench.py --scheme residual --steps 5 --warmup 3 --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 > /dev/null 2>&1; echo "ncu rc=$?"
