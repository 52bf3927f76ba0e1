# one-launch graph bookkeeping: graph tests + config-1 timing
timeout 1200 python -m pytest tests/test_gpu_weights_pf.py tests/test_cli.py tests/test_gpu_fullsize.py -k "graph or cli or strict or every_step" -m "gpu or not gpu" -q -p no:randomly > gpurun_out/g35_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g35_pytest.log
for i in 1 2 3; do timeout 300 python tools/bench_config1.py; done
