#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_rscan_gpu.py -q -m gpu -x -k "large or config5" 2>&1 | tail -25 | tee gpurun_out/big.txt
