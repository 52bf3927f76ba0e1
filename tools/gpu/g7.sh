python -c "from paper_1306_5583_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_resample.py tests/test_gpu_edges.py tests/test_gpu_weights_pf.py tests/test_gpu_gmm.py tests/test_gpu_dist.py -x -q -p no:randomly > gpurun_out/pytest_rs.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_rs.log
B="python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e --no-gmm --no-schemes"
for r in 1 2; do bash tools/ab_lib.sh "$B | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"ms_per_step\"],4), d[\"phase_ms\"], d[\"resample_copy\"][\"ms\"], d[\"gpu_launches\"])'" A OLD; done
bash tools/ab_lib.sh "python tools/bench_gmm.py --seeds 1 2>/dev/null | tail -1 | cut -c1-300" A OLD
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_rs_" -c 40 --csv --log-file gpurun_out/launches_rs.csv python tools/prof_step.py 16777216 6 > /dev/null 2>&1
