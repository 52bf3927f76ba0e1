# one-launch lse reduction: weight / PF / dist / GMM / user tests + step A/B against HEAD
timeout 1800 python -m pytest tests/test_gpu_weights_pf.py tests/test_gpu_dist.py tests/test_gpu_dist_sampler.py tests/test_gpu_gmm.py tests/test_gpu_user.py tests/test_gpu_bench_multirank.py tests/test_gpu_edges.py tests/test_abi.py -m "gpu or not gpu" -q -x -p no:randomly > gpurun_out/g31_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g31_pytest.log
for r in 1 2; do for v in head cur; do
  if [ $v = head ]; then export SMC_LIB_PATH=tools/gpu/head/libsmcb200.so; else unset SMC_LIB_PATH; fi
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e --no-config1 --no-schemes > gpurun_out/g31_$v$r.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/g31_$v$r.json').read().strip().splitlines()[-1]);print('$v$r',round(d['ms_per_step'],4),d['phase_ms'])"
done; done
unset SMC_LIB_PATH
timeout 600 python tools/bench_config1.py > gpurun_out/g31_config1.json 2>&1; cat gpurun_out/g31_config1.json
