# Launch list of the timed step only (NVTX range), then summaries.  1 GPU.
mkdir -p gpurun_out
AXONN_NVTX=1 timeout 1200 ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --no-cpu-baseline --e2e-steps 1 --steps 1 --warmup 3 > gpurun_out/ncu_launch_step.log 2>&1; echo "ncu exit $?"; tail -3 gpurun_out/ncu_launch_step.log
python scripts/ncu_launch_summary.py gpurun_out/launches_step.csv gpurun_out/launch_summary 0 > gpurun_out/launch_summary.log 2>&1; head -40 gpurun_out/launch_summary.log
