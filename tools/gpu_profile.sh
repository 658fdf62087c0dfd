#!/bin/bash
# One GPU session for the judged evidence (run under gpurun from the repo root):
# default bench line, the ncu launch list of the same bench command, and one
# full ncu capture of the checkerboard sweep kernel (config 2, 2000 sweeps).
# Outputs land in gpurun_out/; copy the summaries into profiles/.
set -x
tag=${1:-r01}
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -3 gpurun_out/${tag}_bench.err
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/${tag}_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/${tag}_ncu_launch.log 2>&1
python tools/prof_checker.py 100 100 1024 2000 > gpurun_out/${tag}_p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:checker_sweep -s 1 -c 1 \
    -o gpurun_out/${tag}_checker_c2 python tools/prof_checker.py 100 100 1024 2000 \
    > gpurun_out/${tag}_ncu_full.log 2>&1
tail -2 gpurun_out/${tag}_ncu_full.log
