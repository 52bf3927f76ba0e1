cmd='timeout 300 python bench.py --steps 300 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d[\"phase_ms\"][\"move\"],4), round(d[\"ms_per_step\"],4))"'
bash tools/ab_lib.sh "$cmd" ${VARIANTS:-A O A O A O}
