# ncu --set full of the multinomial scatter / count kernels in the PF step at 2^24 (PF weights)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mn2 -s 6 -c 2 -o gpurun_out/mn2_full python bench.py --steps 4 --warmup 3 --scheme multinomial --no-cpu-baseline --no-gmm --no-schemes --no-e2e --no-config1 > gpurun_out/g39_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/g39_ncu.log
