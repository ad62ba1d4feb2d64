#!/bin/bash
# ncu --set full of the rank-32 fused imputation + selection kernel at C2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"als_select" -c 1 -f \
    -o gpurun_out/c2_select python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_select.log 2>&1
tail -2 gpurun_out/ncu_select.log
