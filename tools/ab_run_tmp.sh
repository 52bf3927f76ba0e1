#!/bin/bash
python bench.py > gpurun_out/r1b_bench.json 2> gpurun_out/r1b_bench.err
python bench.py --impl reference > gpurun_out/r1b_bench_ref.json 2> gpurun_out/r1b_bench_ref.err
A="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-gmm"
python bench.py $A > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b_launches.csv python bench.py $A > gpurun_out/ncu_l.log 2>&1
python tools/prof_step.py 16777216 4 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_pf_move|k_rs_|k_lse" -s 18 -c 9 -o gpurun_out/r1b_full python tools/prof_step.py 16777216 4 > gpurun_out/ncu_full.log 2>&1
