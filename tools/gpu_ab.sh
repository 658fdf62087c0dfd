GSB_CHECKER_GATE=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_api_gpu.py -q -m gpu -x -k "checker or threshold or edge or random" 2>&1 | tail -2
timeout 600 python tools/ab_env.py 100 100 1024 2000 - GSB_CHECKER_GATE=1 - GSB_CHECKER_GATE=1
timeout 600 python tools/ab_env.py 100 100 1024 10000 - GSB_CHECKER_GATE=1
