# 4 GPUs: A8 k sweep at the 12B 2x2 grid (offload off / on), 12B 4x1 offload at the paper's
# per-replica batch (m 256 = 2048 samples, PAPER.md:831-833 weak-scaling batch 16384 / G_data 8)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c13_build.log 2>&1
run() { port=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 "$@"; }
p=29900
for k in 1 2 4 8 16; do p=$((p+1)); run $p --g-inter 2 --coarsen-k $k > gpurun_out/c13_k${k}_off0.jsonl 2>> gpurun_out/c13_bench.err; done
for k in 1 4 16; do p=$((p+1)); run $p --g-inter 2 --coarsen-k $k --offload 1 > gpurun_out/c13_k${k}_off1.jsonl 2>> gpurun_out/c13_bench.err; done
p=$((p+1)); run $p --offload 1 --mb-per-replica 256 --steps 3 --warmup 3 > gpurun_out/c13_4x1_off1_m256.jsonl 2>> gpurun_out/c13_bench.err
echo done
