import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2602_03067_b200 as fsk
n = m = int(sys.argv[1]); d = 64
z = fsk.rng_normal(1001, (n + m) * d)
X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
eng.set_eps(0.05)
f = torch.empty(n, dtype=torch.float32, device="cuda"); g = torch.empty(m, dtype=torch.float32, device="cuda")
eng.bind(f.data_ptr(), g.data_ptr()); eng.init_potentials()
for it in range(6):
    for side, r in ((0, n), (1, m)):
        t0 = time.time(); eng.half_step(side, 0, r); torch.cuda.synchronize()
        print(f"it {it} side {side} {1e3*(time.time()-t0):.1f} ms live {eng.live_set_fraction(side):.3f}", flush=True)
