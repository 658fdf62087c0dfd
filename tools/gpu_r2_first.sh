#!/bin/bash
# round 2, first GPU session: tests, random-scan rates, ncu of rscan2_kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -8 > gpurun_out/gputests.txt; cat gpurun_out/gputests.txt
timeout 600 python tools/rates.py simulated_annealing_random_scan 2>&1 | tee gpurun_out/rates_rscan.txt
python tools/prof_checker.py 100 100 1024 200 simulated_annealing_random_scan > gpurun_out/plain_rs.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rscan2 -s 1 -c 1 -o gpurun_out/prof_rs2 \
  python tools/prof_checker.py 100 100 1024 200 simulated_annealing_random_scan > gpurun_out/ncu_rs2.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_rs2.ncu-rep 40 > gpurun_out/prof_rs2.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_rs2.ncu-rep 60 > gpurun_out/prof_rs2.lines.txt 2>&1
cat gpurun_out/prof_rs2.txt | head -30
