#!/bin/bash
# On a GPU box: the c2 bench line, its launch list and ncu captures of the
# top kernels, into gpurun_out/ (summarise with tools/launch_summary.py and
# tools/ncu_brief.py, then copy the summaries into profiles/).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"als_(seg|mma)_gram" -c 2 -f \
    -o gpurun_out/c2_gram python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:als_select -c 1 -f \
    -o gpurun_out/c2_select python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -8
