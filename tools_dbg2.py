import sys, os
sys.path.insert(0, '.')
import lpfem_inputs as I
from paper_2311_05170_b200 import LPFEM
for ov in (True, False):
    if not ov: os.environ["LPFEM_NO_OVERLAP"] = "1"
    sim = LPFEM(I.config(1))
    for n in range(3):
        try:
            sim.step(); print(ov, n, "ok", sim.stats()["coarse_iters"])
        except Exception as e:
            print(ov, n, "FAIL", e)
    sim.close()
