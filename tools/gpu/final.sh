set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly --durations=15 > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python tools/capture_profiles.py --commit 45222c1dedae > gpurun_out/capture.log 2>&1; echo "capture rc=$?"; cp profiles/move_ncu.json profiles/gmm_mh_ncu.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo "ref rc=$?"
timeout 900 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --no-gmm --no-schemes > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 600 python tools/bench_config1.py > gpurun_out/config1.json 2>&1; echo "c1 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gmm --no-schemes --no-e2e > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?"
