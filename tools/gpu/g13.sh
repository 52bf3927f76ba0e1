python -c "from paper_1306_5583_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e --no-gmm --no-schemes"
for r in 1 2; do bash tools/ab_lib.sh "$B | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"ms_per_step\"],4), d[\"phase_ms\"], d[\"resample_copy\"][\"ms\"], d[\"gpu_launches\"])'" A NOTRIG; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_mn2_count" -s 1 -c 1 -o gpurun_out/mn2_full -f python tools/prof_multinomial.py > gpurun_out/ncu_mn2.log 2>&1; echo ncu rc=$?
