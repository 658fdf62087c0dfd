import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import oracle as O
from paper_2505_18508_b200 import TorusSpec, generate_torus
from paper_2505_18508_b200.campaign import mix_seeds
from paper_2505_18508_b200.solvers import *
O.build()
for (R,C,s) in [(4,4,1),(8,8,42),(50,100,1)]:
    inst=generate_torus(TorusSpec(R,C,s)); w=inst.torus_weights
    seeds=mix_seeds(20250814, range(6))
    for kind in (GREEDY_CHECKERBOARD, ANNEALING_CHECKERBOARD):
        for S in (1,2,3,5,10):
            cfg=default_config(kind,S,0)
            b=run_trials(inst,cfg,seeds)
            bc,bs,se=O.run_trials_checker(R,C,w,kind,S,seeds,cfg.temp_start,cfg.temp_end)
            hx=[b.hex(i)==O.encode_hex(bs[i]) for i in range(6)]
            print(R,C,kind,S,'cut',list(b.best_cut)==list(bc),'se',list(b.sweeps_executed)==list(se),'hex',hx, b.hex(0)[:16], O.encode_hex(bs[0])[:16])
