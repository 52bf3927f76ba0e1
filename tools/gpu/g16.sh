python -c "from paper_1306_5583_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_weights_pf.py -x -q -p no:randomly -k "warp_specialized or full_run or graph or uniform" > gpurun_out/pytest_ws.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_ws.log
timeout 600 python tools/ab_move_ws.py
