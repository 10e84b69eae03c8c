# 1 GPU: 1.3B batch 64 as b_m 64 x 1 / 32 x 2 / 16 x 4 on one box (G_inter = 1: the split only
# trades GEMM size against the A8 overlap of the last backward)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c34_build.log 2>&1
for r in 1 2; do
for mb in "64 1" "32 2" "16 4"; do
  set -- $mb
  timeout 600 python bench.py --no-cpu-baseline --microbatch $1 --mb-per-replica $2 >> gpurun_out/c34_b13_$1x$2.jsonl 2>> gpurun_out/c34_bench.err
done
done
echo done
