python tools/rs2_probe.py 100 100 1024 3000 0 0 7 2 8 2 4 4 2 7 2>&1 | cut -c1-90
python tools/rs2_probe.py 100 140 4096 600 0 0 7 3 4 5 8 3 4 7 2>&1 | cut -c1-90
python tools/rs2_probe.py 100 200 8192 300 0 0 7 4 8 4 4 7 7 5 2>&1 | cut -c1-90
