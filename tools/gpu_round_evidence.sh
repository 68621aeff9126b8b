# Round evidence: bench lines (C2 default, C3, C4), the ncu launch list of the C2
# timed region and one full ncu capture of the attention kernel inside the step.
set -x
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log > gpurun_out/bench_c2.json
timeout 900 python bench.py --config c3 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log > gpurun_out/bench_c3.json
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log > gpurun_out/bench_c4.json
bash tools/prof_r01.sh
ls -la gpurun_out/
