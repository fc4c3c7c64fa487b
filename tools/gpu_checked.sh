# The GPU parity suite against the checked build (device bounds checks, SNN_DCHECK; compute-sanitizer is
# closed on this pool): python -m paper_1903_02440_b200.build --checked, then every -m gpu test with
# SNN_LIB pointing at libsnn_checked.so.  A failed check prints "SNN_CHECKED file:line: condition" and
# traps the launch (the test fails).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python -m paper_1903_02440_b200.build --checked > gpurun_out/build_checked.log 2>&1 || exit 1
SNN_LIB=$PWD/paper_1903_02440_b200/libsnn_checked.so timeout 1500 python -m pytest tests -q -m gpu \
    --ignore=tests/test_gpu_bench_smoke.py > gpurun_out/pytest_checked.log 2>&1; echo checked=$?
tail -3 gpurun_out/pytest_checked.log; grep -c "SNN_CHECKED" gpurun_out/pytest_checked.log
