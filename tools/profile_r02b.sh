#!/bin/bash
# Round-2 re-profile after the c2-ncf / c0xn kernel changes: launch list of the default
# bench command, ncu --set full of the c2-ncf dense kernel (full C2) and of the per-app
# kernel (c0xn, 592 apps = 4 CTAs/SM... one wave), summarised with tools/ncu_brief.py.
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1
OCG_ROWS=1000000 OCG_REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:ncf_fast_kernel \
    -c 1 -f -o gpurun_out/r02b_c2ncf_fast python tools/profile_ncf.py > gpurun_out/r02b_ncu_fast.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ncf_app_batch_kernel -c 1 -f \
    -o gpurun_out/r02b_c0xn python bench.py --workload c0xn --apps 444 --steps 1 --warmup 0 --no-cpu-baseline \
    > gpurun_out/r02b_ncu_c0xn.log 2>&1
python tools/ncu_brief.py gpurun_out/r02b_c2ncf_fast.ncu-rep > gpurun_out/r02b_c2ncf_fast_brief.txt 2>&1
python tools/ncu_brief.py gpurun_out/r02b_c0xn.ncu-rep > gpurun_out/r02b_c0xn_brief.txt 2>&1
python tools/ncu_lines.py gpurun_out/r02b_c0xn.ncu-rep --top 30 > gpurun_out/r02b_c0xn_lines.txt 2>&1
python tools/ncu_lines.py gpurun_out/r02b_c2ncf_fast.ncu-rep --top 30 > gpurun_out/r02b_c2ncf_lines.txt 2>&1
ls -la gpurun_out/
