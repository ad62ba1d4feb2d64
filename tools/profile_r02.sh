#!/bin/bash
# Round-2 profiling run on the GPU box (gpurun): the default bench line and its
# reference arm, the launch list of the default command, ncu captures of the
# dominant c2-ncf kernel (full C2 size) and of the joint-fit epoch kernel.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1
OCG_ROWS=1000000 OCG_REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:ncf_fast_kernel \
    -c 1 -f -o gpurun_out/r02_c2ncf_fast python tools/profile_ncf.py > gpurun_out/r02_ncu_fast.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:joint_epoch_kernel -c 1 -f \
    -o gpurun_out/r02_joint_epoch python tools/profile_joint.py 2 0 1 > gpurun_out/r02_ncu_joint.log 2>&1
