#!/bin/bash
# ncu --set full of the rank-32 half-sweep kernels (row launch of each) at C2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"als_(seg|mma)_gram|als_solve_records" -c 2 -f \
    -o gpurun_out/c2_gram python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_gram.log 2>&1
tail -3 gpurun_out/ncu_gram.log
ls -la gpurun_out/*.ncu-rep
