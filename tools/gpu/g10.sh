python -c "from paper_1306_5583_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/prof_multinomial.py > gpurun_out/mn_plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_mn2_count" -s 1 -c 1 -o gpurun_out/mn2_full -f python tools/prof_multinomial.py > gpurun_out/ncu_mn2.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_mn2.log
