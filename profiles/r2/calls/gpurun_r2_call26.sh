# 1 GPU: calibration of the stage-split cost model at the 12B shape: one stage holding
# embedding + L layers + LN_f / head for L = 2 and 4 (per-layer time from the difference,
# head from the rest; per-shape profile of the head GEMMs)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c26_build.log 2>&1
for L in 2 4; do
  timeout 600 python bench.py --config gpt12b --layers $L --no-cpu-baseline --steps 4 --warmup 3 > gpurun_out/c26_b12_L$L.jsonl 2>> gpurun_out/c26_bench.err
done
echo done
