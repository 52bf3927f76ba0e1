# ncu --set full of one k_pf_move launch (uniform-count, gathering, monitor) at N = 2^24 at the current sources
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pf_move -s 5 -c 1 -o gpurun_out/move_full_r2 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 > gpurun_out/g46_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/g46_ncu.log
