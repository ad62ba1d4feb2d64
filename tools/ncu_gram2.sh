#!/bin/bash
# ncu --set full of the rank-32 Gram kernel: row launch (0) and column launch (1)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"als_mma_gram" -c 2 -f \
    -o gpurun_out/c2_gram2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_gram2.log 2>&1
tail -2 gpurun_out/ncu_gram2.log
