#!/bin/bash
# K4 solver A/B: tests, then c2 with the register-row solver and with OCG_SOLVE_STAGED=1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_als.py tests/test_gpu_multishard.py -x -q > gpurun_out/pytest_als.log 2>&1
rc=$?; echo rc=$rc >> gpurun_out/pytest_als.log; tail -3 gpurun_out/pytest_als.log
[ $rc -ne 0 ] && exit $rc
timeout 240 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
OCG_SOLVE_STAGED=1 timeout 240 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_staged.json 2> gpurun_out/bench_c2_staged.err
python -c "
import json
for f in ['gpurun_out/bench_c2.json','gpurun_out/bench_c2_staged.json']:
    d=json.load(open(f)); print(f, d['ms_per_step'], d['e2e']['value'], d['phases_ms_per_step'])"
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:solve --csv --log-file gpurun_out/launches_solve.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_solve.csv 2>&1 | head -5
