# per-CTA %globaltimer traces of the small attention cases (tools/attn_bench.py)
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for v in ${TRACE_VARIANTS:-0}; do
MIRAGE_ATTN_VARIANT=$v MIRAGE_ATTN_TRACE=1 MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 --reps 10 | sed "s/^/{\"variant\": $v, \"r\": /; s/\$/}/" >> gpurun_out/trace.jsonl
done
