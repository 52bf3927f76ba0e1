# config-5 microbenchmark (all schemes x weight families, 2^10..2^30)
timeout 2400 python tools/bench_resample.py --out gpurun_out/r2_resample_microbench.jsonl > gpurun_out/g21.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/g21.log
