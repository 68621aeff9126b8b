# A/B of the split-combine experiment bits (MIRAGE_ATTN_FOLD) on the small attention cases
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for f in 1 5 3 7; do
MIRAGE_ATTN_FOLD=$f MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama70b_tp8_64x4k --reps 10 | sed "s/^/{\"fold\": $f, \"r\": /; s/\$/}/" >> gpurun_out/fold_trace.jsonl
done
