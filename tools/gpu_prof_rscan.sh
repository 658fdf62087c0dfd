cat > /tmp/rs1.py <<'PY'
import sys, torch; sys.path.insert(0, '.')
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import default_config, run_trials_device
inst = generate_torus(TorusSpec(100, 100, 1)); cfg = default_config("simulated_annealing_random_scan", 200, 0)
run_trials_device(inst, cfg, mix_seeds(20250814, range(1024))); torch.cuda.synchronize(); print("ok")
PY
GSB_RSCAN_BS=$BS python /tmp/rs1.py && GSB_RSCAN_BS=$BS timeout 600 ncu --set full --clock-control none --import-source on -k regex:rscan -c 1 -o gpurun_out/prof_rs python /tmp/rs1.py > gpurun_out/ncu_rs.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_rs.ncu-rep > gpurun_out/prof_rs.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_rs.ncu-rep 40 > gpurun_out/prof_rs.lines.txt 2>&1
rm -f gpurun_out/prof_rs.ncu-rep
