#!/bin/bash
# launch list of the bench command and one full ncu capture of rscan2_kernel at config 2
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-secondary > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_checker.py 100 100 1024 10000 simulated_annealing_random_scan > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rscan2 -s 1 -c 1 \
    -o gpurun_out/prof_rs2 python tools/prof_checker.py 100 100 1024 10000 simulated_annealing_random_scan > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
python tools/ncu_summary.py gpurun_out/prof_rs2.ncu-rep 40 > gpurun_out/prof_rs2.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_rs2.ncu-rep 70 > gpurun_out/prof_rs2.lines.txt 2>&1
head -22 gpurun_out/prof_rs2.txt
