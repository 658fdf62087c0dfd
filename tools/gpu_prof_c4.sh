# ncu full capture of the checkerboard kernel at config 4 (100x200, 8192 trials, 100 sweeps)
set -x
python tools/prof_checker.py 100 200 8192 100 > gpurun_out/c4p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:checker_sweep -s 1 -c 1 \
    -o gpurun_out/prof_c4 python tools/prof_checker.py 100 200 8192 100 > gpurun_out/c4ncu.log 2>&1
tail -2 gpurun_out/c4ncu.log
