# ncu full capture of the attention kernel in the microbench (1 GPU)
CASE=${1:-opt13b_b400}
OUT=${2:-gpurun_out/attn_mb}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_attention -s 3 -c 1 \
  -o $OUT python tools/attn_bench.py --case $CASE --reps 2 > ${OUT}.log 2>&1
tail -2 ${OUT}.log
