#!/bin/bash
# bench.py smoke over its other code paths (development check)
mkdir -p gpurun_out
for args in "--config c5 --sweeps 20 --trials 7 --steps 1 --warmup 1 --no-cpu" \
            "--config c1 --kind simulated_annealing --sweeps 100 --steps 1 --warmup 1 --no-cpu --no-secondary" \
            "--config c1 --kind greedy_random_scan --sweeps 100 --steps 1 --warmup 1 --no-cpu" \
            "--config c2 --kind simulated_annealing_checkerboard --sweeps 500 --steps 1 --warmup 1 --no-cpu --no-secondary"; do
  echo "== bench.py $args"
  python bench.py $args 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print({k:d[k] for k in ('value','n_gpus','gpu_launches')}, d['config']['kind'], d['roofline']['bound'], round(d['roofline']['frac'],4), d['roofline']['kernel'], d['e2e'] and round(d['e2e']['value']/d['value'],3))"
done 2>&1 | tee gpurun_out/bench_variants.txt
