python tools/rs2_probe.py 100 140 4096 600 0 0 9 2 4 5 2>&1 | cut -c1-90
python tools/rs2_probe.py 100 200 8192 300 0 0 13 2 7 4 2>&1 | cut -c1-90
python tools/rs2_probe.py 100 100 1024 3000 0 0 2>&1 | cut -c1-90
python tools/rs2_probe.py 50 100 100 1000 0 0 2>&1 | cut -c1-90
