# round-end records on one box: GPU suite, smoke, profile capture (stamped with the source hash), the bench
# line, the reference arm, config 4 on one GPU, config-5 microbenchmark, launch list.  $1 = commit label.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly --durations=15 > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python tools/capture_profiles.py --commit "$1" > gpurun_out/capture.log 2>&1; echo "capture rc=$?"; cp profiles/move_ncu.json profiles/gmm_mh_ncu.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo "ref rc=$?"
timeout 900 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --no-gmm --no-schemes --no-config1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 2400 python tools/bench_resample.py --out gpurun_out/resample_microbench.jsonl > gpurun_out/mb.log 2>&1; echo "mb rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?"
