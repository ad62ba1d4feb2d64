#!/bin/bash
# every bench workload once (1 GPU), JSON lines into gpurun_out/
mkdir -p gpurun_out
for w in c1 c0xn ingest; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?"; head -c 400 gpurun_out/bench_$w.json; echo
done
