# zsp/scan1 single-pass scans: resample + dist + fullsize tests, A/B vs the round-2 commit library, launch list
set -x
timeout 1200 python -m pytest tests/test_gpu_resample.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py tests/test_gpu_dist_sampler.py -m gpu -q -x -p no:randomly > gpurun_out/g20_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g20_pytest.log
for i in 1 2; do for v in old new; do
  if [ $v = old ]; then export SMC_LIB_PATH=tools/gpu/old/libsmcb200.so; else unset SMC_LIB_PATH; fi
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e --no-schemes > gpurun_out/g20_$v$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/g20_$v$i.json').read().strip().splitlines()[-1]);print('$v$i',round(d['ms_per_step'],4),d['phase_ms'])"
done; done
unset SMC_LIB_PATH
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/g20_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmm --no-schemes --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
