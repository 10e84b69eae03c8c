# 4 GPUs: stage split from measured busy times (reading D-21d, bench --stage-balance 3) vs the
# FLOP split, 12B 4x1 48 layers (the N = 4 default) and the 16-layer sweep point
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c30_build.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29881 bench.py --gpus 4 --stage-balance 3 > gpurun_out/c30_n4_sb3.jsonl 2> gpurun_out/c30_bench.err
timeout 900 $R --master-port 29882 bench.py --gpus 4 > gpurun_out/c30_n4_sb1.jsonl 2>> gpurun_out/c30_bench.err
timeout 900 $R --master-port 29883 bench.py --gpus 4 --config gpt12b --layers 16 --g-inter 4 --mb-per-replica 64 --steps 4 --stage-balance 3 > gpurun_out/c30_16l_sb3.jsonl 2>> gpurun_out/c30_bench.err
echo done
