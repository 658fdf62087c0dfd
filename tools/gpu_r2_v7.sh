#!/bin/bash
# round 2, kernel v7 (sweep slices): launch list, full ncu capture, other configs' bench lines
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-secondary > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
python tools/prof_checker.py 100 100 1024 10000 simulated_annealing_random_scan > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rscan2 -s 1 -c 1 \
    -o gpurun_out/prof_rs2 python tools/prof_checker.py 100 100 1024 10000 simulated_annealing_random_scan > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
python tools/ncu_summary.py gpurun_out/prof_rs2.ncu-rep 40 > gpurun_out/prof_rs2.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_rs2.ncu-rep 70 > gpurun_out/prof_rs2.lines.txt 2>&1
head -22 gpurun_out/prof_rs2.txt
for c in c1 c3 c5; do
  python bench.py --config $c --steps 3 --warmup 3 --no-secondary > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; cut -c1-200 gpurun_out/bench_$c.json
done
python bench.py --config c4 --steps 2 --warmup 3 --no-secondary > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cut -c1-200 gpurun_out/bench_c4.json
