# 4 GPUs: where the 4x1 bubble above (P-1)/(m+P-1) comes from: per-op timelines of every
# stage (AXONN_TIMELINE) at the 16-layer sweep point, and the speed-calibrated split (D-21c)
mkdir -p gpurun_out/c29_tl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c29_build.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
AXONN_TIMELINE=gpurun_out/c29_tl/gi4 timeout 900 $R --master-port 29871 bench.py --gpus 4 --config gpt12b --layers 16 --g-inter 4 --mb-per-replica 64 --steps 4 > gpurun_out/c29_gi4.jsonl 2> gpurun_out/c29_bench.err
timeout 900 $R --master-port 29872 bench.py --gpus 4 --config gpt12b --layers 16 --g-inter 4 --mb-per-replica 64 --steps 4 --stage-balance 2 > gpurun_out/c29_gi4_cal.jsonl 2>> gpurun_out/c29_bench.err
echo done
