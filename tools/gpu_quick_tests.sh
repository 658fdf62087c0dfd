#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_distributed_gpu.py tests/test_api_gpu.py -q -m gpu -x 2>&1 | tail -8 | tee gpurun_out/quick.txt
