# 2 GPUs: the fp16 build (N2: static loss scale 1024, overflow skip) on the driver's N = 1 and
# N = 2 workloads; the reference arm under torchrun (rank 0 prints, the other rank exits 0)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c35_build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --dtype fp16 > gpurun_out/c35_b13_fp16.jsonl 2> gpurun_out/c35_bench.err
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29901 bench.py --gpus 2 --dtype fp16 > gpurun_out/c35_b12_2x1_fp16.jsonl 2>> gpurun_out/c35_bench.err
timeout 600 $R --master-port 29902 bench.py --gpus 2 --impl reference --steps 2 --warmup 3 > gpurun_out/c35_ref_n2.jsonl 2>> gpurun_out/c35_bench.err; echo "ref n2 exit $?" >> gpurun_out/c35_bench.err
echo done
