#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_als.py tests/test_gpu_multishard.py -x -q > gpurun_out/pytest_als.log 2>&1
rc=$?; echo rc=$rc >> gpurun_out/pytest_als.log; tail -3 gpurun_out/pytest_als.log
[ $rc -ne 0 ] && exit $rc
timeout 240 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "
import json
for f in ['gpurun_out/bench_c2.json','gpurun_out/bench_c3.json']:
    d=json.load(open(f)); print(f, d['ms_per_step'], d['e2e']['value'], d['phases_ms_per_step'], d['roofline']['frac'])"
