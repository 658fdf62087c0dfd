set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err; tail -3 gpurun_out/s1_bench.err; cat gpurun_out/s1_bench.json
timeout 600 python tools/team_sweep.py 100x100x1024x2000 100x140x4096x500 100x200x8192x250 2>&1 | tail -4
timeout 900 python bench.py --config c5 --steps 3 > gpurun_out/s1_c5.json 2> gpurun_out/s1_c5.err; tail -3 gpurun_out/s1_c5.err; cat gpurun_out/s1_c5.json
