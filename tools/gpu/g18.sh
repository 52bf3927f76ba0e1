# k_rs_scan1 A/B: resample tests, then interleaved bench runs old/new lib on the same box
set -x
timeout 900 python -m pytest tests/test_gpu_resample.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:randomly > gpurun_out/g18_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g18_pytest.log
for i in 1 2 3; do
  SMC_LIB_PATH=tools/gpu/old/libsmcb200.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e > gpurun_out/g18_old_$i.json 2>/dev/null
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e > gpurun_out/g18_new_$i.json 2>/dev/null
done
python - <<'P'
import json
for t in ("old","new"):
    for i in (1,2,3):
        d=json.loads(open(f"gpurun_out/g18_{t}_{i}.json").read().strip().splitlines()[-1])
        print(t,i,round(d["ms_per_step"],4), d.get("phase_ms"), json.dumps(d.get("schemes"))[:600])
P
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/g18_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmm --no-schemes --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
