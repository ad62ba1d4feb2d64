#!/bin/bash
# one full ncu capture of the first row-side K4 solver launch of a c2 step
mkdir -p gpurun_out
K=${1:-als_solve}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 -f \
    -o gpurun_out/c2_solve python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
