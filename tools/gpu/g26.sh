# full GPU suite + bench (current) + PF scheme sweep of the pre-today library for comparison
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly --durations=10 > gpurun_out/g26_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/g26_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g26_bench.json 2> gpurun_out/g26_bench.err; echo "bench rc=$?"
SMC_LIB_PATH=tools/gpu/old/libsmcb200.so timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gmm --no-e2e --no-config1 > gpurun_out/g26_bench_old.json 2> gpurun_out/g26_bench_old.err; echo "bench old rc=$?"
python - <<'P'
import json
for f in ("g26_bench","g26_bench_old"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["ms_per_step"],4), {k:round(v["ms_per_step"],4) for k,v in d.get("schemes",{}).items()}, d.get("config1"), (d.get("cpu_baseline") or {}).get("config1"))
P
