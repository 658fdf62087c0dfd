#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/rscan_stress.py 150 33 2>&1 | tail -3
python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -2 gpurun_out/bench_c5.err; cut -c1-300 gpurun_out/bench_c5.json
