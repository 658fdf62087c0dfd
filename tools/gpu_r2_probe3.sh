#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_rscan_gpu.py -q -m gpu -x 2>&1 | tail -15 | tee gpurun_out/rs_tests.txt
{
python tools/rs2_probe.py 100 100 1024 1000 0 0 2 7 4 4 8 2
python tools/rs2_probe.py 100 100 1024 10000 0 0
GSB_LIB=build_variants/libgsb_prof.so python tools/rs2_probe.py 100 100 1024 10000 0 0
python tools/rs2_probe.py 100 140 4096 300 0 0 4 5 8 3
python tools/rs2_probe.py 100 200 8192 100 0 0 4 7 8 4
python tools/rs2_probe.py 50 100 100 1000 0 0 8 1 4 2 2 4
} 2>&1 | tee gpurun_out/rs2_probe3.txt
