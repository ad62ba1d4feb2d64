#!/bin/bash
# On a GPU box: the default (c2) bench line, the reference arm, the launch list
# of the default command and ncu --set full captures of the hot kernels, into
# gpurun_out/ (summarise with tools/launch_summary.py, tools/ncu_brief.py,
# tools/ncu_lines.py; copy the summaries into profiles/).
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_c2_reference.json 2> gpurun_out/bench_c2_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"als_mma_gram" -c 2 -f \
    -o gpurun_out/c2_gram python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"als_solve" -c 1 -f \
    -o gpurun_out/c2_solve python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"als_select" -c 1 -f \
    -o gpurun_out/c2_select python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -12
