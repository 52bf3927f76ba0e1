python -c "from paper_1306_5583_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_pf_move_ws" -s 4 -c 1 -o gpurun_out/ws_full -f python tools/prof_step.py 16777216 6 > gpurun_out/ncu_ws.log 2>&1; echo ncu rc=$?
