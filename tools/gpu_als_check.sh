#!/bin/bash
# ALS GPU tests, then (only if they pass) the default bench line and its launch list
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_als.py tests/test_gpu_multishard.py -x -q > gpurun_out/pytest_als.log 2>&1
rc=$?; echo rc=$rc >> gpurun_out/pytest_als.log
tail -30 gpurun_out/pytest_als.log
[ $rc -ne 0 ] && exit $rc
timeout 240 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c2.csv 2>&1 | head -20
