import sys, numpy as np
sys.path.insert(0, '.')
import lpfem_inputs as I
from oracle import alg3
from paper_2311_05170_b200 import LPFEM, build
build.build()
def cmp(cfg, steps=1):
    ora = alg3.Alg3(cfg); sim = LPFEM(cfg)
    for n in range(steps):
        ora.step(); 
        try:
            sim.step()
        except Exception as e:
            print("STEP FAIL", e, sim.stats()); return
        g, o = sim.fields(), ora.fields()
        gc, oc = sim.coarse_fields(), ora.coarse.state
        for k in ("pF","pf","pm","u","p"):
            print(n+1, k, "fine maxdiff", np.abs(np.ravel(g[k])-np.ravel(o[k])).max(), "max|ora|", np.abs(o[k]).max(),
                  "coarse maxdiff", np.abs(np.ravel(gc[k])-np.ravel(oc[k])).max())
        du = np.abs(g["u"]-o["u"]).max(axis=0); i = int(np.argmax(du)); print("  worst u node", i, ora.Xc[i], g["u"][:, i], o["u"][:, i])
    print(sim.stats())
print("=== constant"); cmp(I.config(0, problem="constant", steps=1))
print("=== injection"); cmp(I.make_config(dim=2, H=1/4, h=1/16, grid=2, dt=0.01, steps=2, problem="injection", seed=2), 2)
print("=== cfg1 1 step no-oracle")
sim = LPFEM(I.config(1), max_iter=200000)
import time; t=time.time()
try:
    sim.step()
except Exception as e:
    print("FAIL", e)
print(time.time()-t, sim.stats())
