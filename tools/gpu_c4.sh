#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_als.py -x -q -k "upload or fused_selection" > gpurun_out/pytest_c4.log 2>&1
rc=$?; echo rc=$rc >> gpurun_out/pytest_c4.log; tail -5 gpurun_out/pytest_c4.log
[ $rc -ne 0 ] && exit $rc
timeout 600 python bench.py --workload c4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
