python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests/test_gpu_attention.py tests/test_gpu_attention_fuzz.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py tests/test_gpu_decode_fuzz.py tests/test_gpu_prefill.py -q -p no:cacheprovider 2>&1 | tail -4
export MIRAGE_ATTN_TRACE=1
python tools/attn_bench.py --case llama70b_tp8_64x4k --reps 30 > gpurun_out/r02_trace6.jsonl 2>&1
unset MIRAGE_ATTN_TRACE
MIRAGE_ATTN_REPEAT=8 python tools/attn_bench.py --case llama3_8b_1x8k llama3_8b_1x32k llama3_8b_4x16k llama3_8b_4x32k llama70b_tp8_64x4k opt13b_b29 opt13b_b400 llama3_8b_32x32k --reps 10 >> gpurun_out/r02_trace6.jsonl 2>&1
MIRAGE_ATTN_REPEAT=8 python tools/attn_bench.py --case llama70b_tp8_64x4k --split 256 512 1024 2048 --reps 10 >> gpurun_out/r02_trace6.jsonl 2>&1
cat gpurun_out/r02_trace6.jsonl | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except: print(l[:200]); continue
    t=d.get('trace',{})
    print(d['case'], d.get('split_blocks'), d.get('units'), d.get('kernel_ms'), round(d.get('gbs_kernel',0)), t)
"
