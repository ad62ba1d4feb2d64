#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"als_solve_records" -c 1 -f \
    -o gpurun_out/c2_solve python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
