#!/bin/bash
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 | tee gpurun_out/gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
