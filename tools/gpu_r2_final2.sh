#!/bin/bash
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -x 2>&1 | tail -6 | tee gpurun_out/gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; cut -c1-200 gpurun_out/bench_c5.json
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
python tools/prof_checker.py 2000 2000 8 100 simulated_annealing_random_scan > gpurun_out/plain_big.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:rscan_big -s 1 -c 1 -o gpurun_out/prof_big python tools/prof_checker.py 2000 2000 8 100 simulated_annealing_random_scan > gpurun_out/ncu_big.log 2>&1; python tools/ncu_summary.py gpurun_out/prof_big.ncu-rep 12 > gpurun_out/prof_big.txt 2>&1; head -20 gpurun_out/prof_big.txt
