# A/B of dev knobs on the checkerboard engine (timings + result digest)
timeout 600 python tools/ab_env.py 100 100 1024 2000 - GSB_CHECKER_WARPS=2 GSB_CHECKER_THIN=1
