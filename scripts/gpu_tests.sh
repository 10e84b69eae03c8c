set -x; mkdir -p gpurun_out
python -c "from paper_2110_13005_b200 import build; build.build()"
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/gpu_tests.log
tail -40 gpurun_out/gpu_tests.log
