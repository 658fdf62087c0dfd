#!/bin/bash
mkdir -p gpurun_out
{
python tools/rs2_probe.py 100 140 4096 300 0 0 2 10 4 7 4 10 2 13
python tools/rs2_probe.py 100 200 8192 100 0 0 2 13 4 7 4 10 4 13
python tools/rs2_probe.py 100 200 2048 300 0 0 2 13 4 7
GSB_LIB=build_variants/libgsb_prof.so python tools/rs2_probe.py 100 200 2048 300 2 13 4 7
} 2>&1 | tee gpurun_out/rs2_probe2.txt
