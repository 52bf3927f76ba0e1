# The GPU suite against the checked build (-DSMC_CHECKED=1: kernel index guards counted, scratch
# workspaces filled with 0xA5 instead of whatever the allocator hands out); after every test the
# conftest fixture asserts that no guard fired.  compute-sanitizer is closed on this pool.
mkdir -p tools/gpu/checked
SMC_LIB_PATH=$PWD/tools/gpu/checked/libsmcb200.so python -c "from paper_1306_5583_b200 import _build; _build.build(force=True, extra=('-DSMC_CHECKED=1',))"
export SMC_LIB_PATH=tools/gpu/checked/libsmcb200.so SMC_CHECKED_RUN=1
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/checked_pytest.log 2>&1; echo "checked pytest rc=$?"; tail -6 gpurun_out/checked_pytest.log
python -c "from paper_1306_5583_b200 import _abi; import torch; print('checked build:', _abi.check_failures())"
