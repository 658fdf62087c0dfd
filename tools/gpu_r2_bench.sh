#!/bin/bash
# round 2 GPU session: bench (default = random scan, config 2), reference arm, launch list,
# full ncu capture of rscan2_kernel at the bench launch, final-cut distributions
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-200 gpurun_out/bench_ref.json
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-secondary > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
python tools/prof_checker.py 100 100 1024 10000 simulated_annealing_random_scan > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rscan2 -s 1 -c 1 \
    -o gpurun_out/prof_rs2 python tools/prof_checker.py 100 100 1024 10000 simulated_annealing_random_scan > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
python tools/ncu_summary.py gpurun_out/prof_rs2.ncu-rep 40 > gpurun_out/prof_rs2.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_rs2.ncu-rep 70 > gpurun_out/prof_rs2.lines.txt 2>&1
head -16 gpurun_out/prof_rs2.txt
timeout 900 python tools/cut_distribution.py 50 100 1024 1000 100 100 4096 10000 100 140 1024 2000 > gpurun_out/cut_distributions.jsonl 2> gpurun_out/cutdist.err; cut -c1-200 gpurun_out/cut_distributions.jsonl
