export SMC_LIB_PATH=$PWD/paper_1306_5583_b200/libsmcb200_OLD.so
timeout 300 python tools/prof_step.py 16777216 8 > gpurun_out/old_plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --set full --clock-control none -k regex:"k_rs_" -s 30 -c 6 -o gpurun_out/rs_old_full -f python tools/prof_step.py 16777216 8 > gpurun_out/ncu_rs_old.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_rs_old.log
