#!/bin/bash
# round 2: random-scan tests, then the bench on every config (full schedules)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_rscan_gpu.py -q -m gpu -x 2>&1 | tail -4
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err; cut -c1-400 gpurun_out/bench_c2.json
python bench.py --config c1 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; cut -c1-300 gpurun_out/bench_c1.json
python bench.py --config c3 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; cut -c1-300 gpurun_out/bench_c3.json
python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cut -c1-300 gpurun_out/bench_c4.json
