# split-size sweep in the small-batch regime (tokens per split; 0 = planner)
python -c "import __graft_entry__ as g; g.build()" >/dev/null
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x8k --split 0 112 80 56 --reps 10 >> gpurun_out/split.jsonl
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_1x32k --split 0 448 304 224 --reps 10 >> gpurun_out/split.jsonl
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama3_8b_4x16k --split 0 912 608 448 --reps 10 >> gpurun_out/split.jsonl
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case llama70b_tp8_64x4k --split 0 512 336 256 --reps 10 >> gpurun_out/split.jsonl
MIRAGE_ATTN_REPEAT=8 timeout 300 python tools/attn_bench.py --case opt13b_b29 --split 0 1024 768 512 --reps 10 >> gpurun_out/split.jsonl
