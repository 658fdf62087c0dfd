#!/bin/bash
# round 2 final GPU session: all GPU tests, smoke, bench (default), reference arm, launch list, ncu
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -x 2>&1 | tail -6 | tee gpurun_out/gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
bash tools/gpu_r2_bench.sh
python bench.py --config c3 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; cut -c1-200 gpurun_out/bench_c3.json
python bench.py --config c1 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; cut -c1-200 gpurun_out/bench_c1.json
python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cut -c1-200 gpurun_out/bench_c4.json
