#!/bin/bash
# One GPU session: tests, bench, launch list, full ncu capture of the sweep kernel.
set -x
python -m pytest tests -q -m gpu 2>&1 | tail -3
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python tools/prof_checker.py 100 100 1024 2000 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:checker_sweep -s 1 -c 1 \
    -o gpurun_out/prof_checker python tools/prof_checker.py 100 100 1024 2000 > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
