# full ncu capture of the attention kernel for a small (latency-bound) case and the C2 case
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_attention -s 3 -c 1 \
  -o gpurun_out/attn_1x32k python tools/attn_bench.py --case llama3_8b_1x32k --reps 2 > gpurun_out/attn_1x32k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_attention -s 3 -c 1 \
  -o gpurun_out/attn_70b python tools/attn_bench.py --case llama70b_tp8_64x4k --reps 2 > gpurun_out/attn_70b.log 2>&1
ls -la gpurun_out
