# launch lists of the multinomial and residual PF steps at 2^24 (where the extra time over systematic goes)
for sc in multinomial residual; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$sc.csv python bench.py --steps 10 --warmup 3 --scheme $sc --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 > /dev/null 2>&1
  echo "== $sc"; python tools/launches.py gpurun_out/launches_$sc.csv
  timeout 300 python bench.py --steps 30 --warmup 5 --scheme $sc --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['phase_ms'])"
done
