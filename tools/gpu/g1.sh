set -x
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:randomly --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"
  tail -5 gpurun_out/san_$t.log
done
