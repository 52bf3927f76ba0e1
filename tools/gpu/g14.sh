python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/capture_profiles.py --commit cd714787c33f > gpurun_out/capture.log 2>&1; echo "capture rc=$?"; tail -c 1500 gpurun_out/capture.log; cp profiles/move_ncu.json profiles/gmm_mh_ncu.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_final.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo "ref rc=$?"
