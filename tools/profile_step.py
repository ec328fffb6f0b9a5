"""One config, a few steps (for ncu captures): python tools/profile_step.py CFG STEPS"""
import sys
sys.path.insert(0, '.')
import lpfem_inputs as I
from paper_2311_05170_b200 import LPFEM
cfg = I.config(int(sys.argv[1]))
sim = LPFEM(cfg)
for _ in range(int(sys.argv[2])):
    sim.step()
print(sim.stats())
