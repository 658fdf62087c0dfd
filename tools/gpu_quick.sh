# parity of the checkerboard engines + quick timings (development loop)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_api_gpu.py tests/test_cluster_gpu.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python tools/quick.py 2>&1 | tail -6
