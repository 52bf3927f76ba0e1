# split move (normals on a side stream): bit identity vs the fused move, PF tests, step A/B
for sp in 0 1; do echo "split=$sp hash $(SMC_PF_SPLIT=$sp PYTHONPATH=. timeout 300 python tools/state_hash.py 1048576 8 2>&1 | tail -1)"; done
for sp in 0 1; do echo "split=$sp hash2e24 $(SMC_PF_SPLIT=$sp PYTHONPATH=. timeout 300 python tools/state_hash.py 16777216 5 2>&1 | tail -1)"; done
timeout 1800 python -m pytest tests/test_gpu_weights_pf.py tests/test_gpu_dist_sampler.py tests/test_gpu_bench_multirank.py tests/test_gpu_fullsize.py -k "not past_shared and not 100_obs_end" -m gpu -q -x -p no:randomly > gpurun_out/g33_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g33_pytest.log
for r in 1 2; do for sp in 0 1; do
  SMC_PF_SPLIT=$sp timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-gmm --no-config1 --no-schemes > gpurun_out/g33_$sp$r.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/g33_$sp$r.json').read().strip().splitlines()[-1]);print('split=$sp r$r',round(d['ms_per_step'],4),d['phase_ms'],'e2e',round(d['e2e']['value']/1e10,4))"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/g33_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 > /dev/null 2>&1; echo "ncu rc=$?"
