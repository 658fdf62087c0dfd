#!/bin/bash
mkdir -p gpurun_out
{
python tools/rs2_probe.py 100 100 1024 1000 0 0 1 13 2 7 4 4 2 4 4 2 4 7
python tools/rs2_probe.py 100 100 1024 10000 0 0 2 7
GSB_LIB=build_variants/libgsb_prof.so python tools/rs2_probe.py 100 100 1024 1000 1 13 2 7 4 4
GSB_LIB=build_variants/libgsb_prof.so python tools/rs2_probe.py 100 100 1024 10000 1 13 2 7
python tools/rs2_probe.py 100 140 4096 300 0 0 2 7 4 4
python tools/rs2_probe.py 100 200 8192 100 0 0 2 7 4 4 2 10
python tools/rs2_probe.py 50 100 100 1000 0 0 2 7 4 4 4 2 4 1
} 2>&1 | tee gpurun_out/rs2_probe.txt
