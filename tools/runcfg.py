"""Run BASELINE config i for k steps on cuda:0 and print per-step timing and solver statistics."""
import json, sys, time
sys.path.insert(0, '.')
import lpfem_inputs as I
from paper_2311_05170_b200 import LPFEM, build
build.build()
i = int(sys.argv[1]); k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = I.config(i)
t0 = time.time()
sim = LPFEM(cfg, max_iter=int(sys.argv[3]) if len(sys.argv) > 3 else 20000)
print(f"cfg{i} create {time.time()-t0:.2f}s", flush=True)
prev = sim.stats()
for n in range(k):
    t = time.time()
    try:
        sim.step()
    except Exception as e:
        print("FAIL", e)
    s = sim.stats()
    print(f"step {n+1}: {time.time()-t:.3f}s coarse {s['t_coarse_ms']-prev['t_coarse_ms']:.1f}ms fine {s['t_fine_ms']-prev['t_fine_ms']:.1f}ms "
          f"pcg {s['t_krylov_ms'][0]-prev['t_krylov_ms'][0]:.1f}ms gmres {s['t_krylov_ms'][1]-prev['t_krylov_ms'][1]:.1f}ms "
          f"iters pcg sum {s['fine_iters'][0]-prev['fine_iters'][0]} max {s['fine_max_iters'][0]} gmres sum {s['fine_iters'][1]-prev['fine_iters'][1]} max {s['fine_max_iters'][1]} "
          f"picard {s['picard_iters']-prev['picard_iters']} res {s['max_rel_residual']} "
          f"bytes_krylov [{s['bytes_krylov'][0]-prev['bytes_krylov'][0]:.4e}, {s['bytes_krylov'][1]-prev['bytes_krylov'][1]:.4e}]", flush=True)
    prev = s
print(json.dumps({k: v for k, v in s.items()}))
