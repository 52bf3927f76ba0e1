# multinomial MN1 path past the shared-memory bins + config-5 microbenchmark
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -k "past_shared" tests/test_gpu_resample.py -m gpu -q -x -p no:randomly > gpurun_out/g22_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g22_pytest.log
timeout 2400 python tools/bench_resample.py --out gpurun_out/r2_resample_microbench.jsonl > gpurun_out/g22_mb.log 2>&1; echo "mb rc=$?"; tail -2 gpurun_out/g22_mb.log
