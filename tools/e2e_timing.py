import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench, paper_2602_03067_b200 as fsk
n, m, d, eps, iters = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
X, Y = bench.make_inputs(n, m, d)
a, b = bench.uniform_weights(n), bench.uniform_weights(m)
for rep in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    out = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=iters, precision="single", grad=True)
    print(f"rep {rep}: {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
