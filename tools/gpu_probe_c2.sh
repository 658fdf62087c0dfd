#!/bin/bash
mkdir -p gpurun_out
{
python tools/rs2_probe.py 100 100 1024 3000 0 0
python tools/rs2_probe.py 100 140 4096 300 0 0
python tools/rs2_probe.py 100 200 8192 100 0 0
python tools/rs2_probe.py 50 100 100 1000 0 0
timeout 900 python -m pytest tests/test_rscan_gpu.py -q -m gpu -x 2>&1 | tail -3
} 2>&1 | tee gpurun_out/probe_c2.txt
