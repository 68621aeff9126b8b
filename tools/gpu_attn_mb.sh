# attention microbench: kernel-only event timing (MIRAGE_FLAG_TIME_ATTN), planner splits, NS variants
set -x
timeout 600 python tools/attn_bench.py --reps 30 > gpurun_out/attn_mb_v0.txt 2>&1
MIRAGE_ATTN_VARIANT=1 timeout 600 python tools/attn_bench.py --reps 30 > gpurun_out/attn_mb_v1.txt 2>&1
timeout 600 python tools/attn_bench.py --reps 20 --case llama3_8b_1x32k llama3_8b_4x16k llama70b_tp8_64x4k opt13b_b29 --split 0 256 512 1024 2048 4096 > gpurun_out/attn_mb_split.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:paged_attention -s 3 -c 3 --csv --log-file gpurun_out/attn_small_ncu.csv python tools/attn_bench.py --reps 3 --case llama3_8b_1x32k llama70b_tp8_64x4k > /dev/null 2>&1
cat gpurun_out/attn_mb_v0.txt gpurun_out/attn_mb_v1.txt
