# K2 diagnostic variants (compile-time AXONN_ATTN_EXP, separate libraries; GPU box)
set -e
mkdir -p gpurun_out
VARS="${ATTN_EXP_VARIANTS:-1 2 4 3}"
for e in $VARS; do
  AXONN_DIAG_DEFINES="-DAXONN_ATTN_EXP=$e" AXONN_DIAG_TAG=_exp$e python -c "from paper_2110_13005_b200 import build; build.build(dtypes=('bf16',))" > /dev/null &
done
wait
for b in ${ATTN_EXP_B:-8 32}; do
  python scripts/attn_bench.py --b $b --tag base
  for e in $VARS; do
    python scripts/attn_bench.py --b $b --tag exp$e --lib paper_2110_13005_b200/libaxonn_exp$e.so
  done
done
