#!/usr/bin/env python3
"""Generates tests/golden/reference_golden.npz from the reference itself.

Runs in the build container only (needs oracle/_ref, i.e. /root/reference
compiled by oracle/build_ref.py). Every output below comes from the
reference's own C++ code path (fsk::stream / fsk::solver), with inputs drawn
from the reference generator (fsk::Rng, restated bit-exactly in oracle/rng.py)
on the shapes of proj/tests/test_stream.cpp plus the BASELINE cfg1 workload.
The committed .npz is the golden vector set the oracle and the GPU tests are
pinned to (the reference ships none: SURVEY.md §4).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import Oracle  # noqa: E402
from oracle.rng import Rng, random_measure  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_golden.npz"


def main():
    ref = Oracle("ref")
    G = {}

    # test_stream.cpp:112 f-update vs dense (n=m=64, d=4, tiles 16x24, simplex weights)
    rng = Rng(101)
    X, a = random_measure(rng, 64, 4, False)
    Y, b = random_measure(rng, 64, 4, False)
    g = rng.normal_vector(64)
    G.update(fu_X=X, fu_a=a, fu_Y=Y, fu_b=b, fu_g=g,
             fu_out=ref.update_f_hat(X, a, Y, b, g, 0.1, (16, 24)))

    # test_stream.cpp:126 g-update (n=23, m=31, d=3, tiles 8x8)
    rng = Rng(17)
    X, a = random_measure(rng, 23, 3, False)
    Y, b = random_measure(rng, 31, 3, False)
    f = rng.normal_vector(23)
    G.update(gu_X=X, gu_a=a, gu_Y=Y, gu_b=b, gu_f=f,
             gu_out=ref.update_g_hat(X, a, Y, b, f, 0.2, (8, 8)))

    # ragged tiles (test_stream.cpp:140 shape), the bug-fixed path
    rng = Rng(23)
    X, a = random_measure(rng, 53, 3, False)
    Y, b = random_measure(rng, 41, 3, False)
    g = rng.normal_vector(41)
    G.update(tl_X=X, tl_a=a, tl_Y=Y, tl_b=b, tl_g=g,
             tl_out=ref.update_f_hat(X, a, Y, b, g, 0.15, (5, 7)))

    # transport ops at rough potentials (test_stream.cpp:200-325 shapes)
    rng = Rng(47)
    X, a = random_measure(rng, 64, 4, False)
    Y, b = random_measure(rng, 64, 4, False)
    sol = ref.sinkhorn_solve(X, a, Y, b, eps=0.3, max_iters=20, tiles=(16, 16))
    fh, gh = sol["f_hat"], sol["g_hat"]
    V = np.array([[rng.normal() for _ in range(3)] for _ in range(64)])
    U = np.array([[rng.normal() for _ in range(2)] for _ in range(64)])
    A = np.array([[rng.normal() for _ in range(2)] for _ in range(64)])
    B = np.array([[rng.normal() for _ in range(2)] for _ in range(64)])
    r, c = ref.induced_marginals(X, a, Y, b, fh, gh, 0.3, (16, 16))
    fs, gs = ref.symmetric_update(X, a, Y, b, fh, gh, 0.3, (7, 9))
    G.update(tr_X=X, tr_a=a, tr_Y=Y, tr_b=b, tr_f=fh, tr_g=gh, tr_V=V, tr_U=U, tr_A=A, tr_B=B,
             tr_PV=ref.apply_plan(X, a, Y, b, fh, gh, 0.3, V, (16, 16)),
             tr_PtU=ref.apply_plan_adjoint(X, a, Y, b, fh, gh, 0.3, U, (5, 6)),
             tr_HV=ref.apply_hadamard_plan(X, a, Y, b, fh, gh, 0.3, A, B, V[:, :2], (8, 8)),
             tr_r=r, tr_c=c, tr_sym_f=fs, tr_sym_g=gs,
             tr_dual=np.array(ref.dual_cost(X, a, Y, b, fh, gh, 0.3, (16, 16))))

    # label-augmented f-update (test_stream.cpp:442)
    rng = Rng(97)
    la = np.array([rng.next_u64() % 3 for _ in range(18)], dtype=np.int32)
    lb = np.array([rng.next_u64() % 3 for _ in range(22)], dtype=np.int32)
    X, a = random_measure(rng, 18, 2)
    Y, b = random_measure(rng, 22, 2)
    W = np.zeros((3, 3))
    W[0, 1] = W[1, 0] = 1.5
    W[0, 2] = W[2, 0] = 0.75
    W[1, 2] = W[2, 1] = 2.25
    g = rng.normal_vector(22)
    cost = dict(lambda1=0.5, lambda2=0.5, label_cost=W)
    G.update(lab_X=X, lab_a=a, lab_Y=Y, lab_b=b, lab_la=la, lab_lb=lb, lab_W=W, lab_g=g,
             lab_out=ref.update_f_hat(X, a, Y, b, g, 0.25, (5, 4), cost=cost, la=la, lb=lb))

    # solver: double/single x alternating/symmetric, tolerance, eps scaling
    rng = Rng(1234)
    X, a = random_measure(rng, 96, 5, False)
    Y, b = random_measure(rng, 80, 5, False)
    G.update(sv_X=X, sv_a=a, sv_Y=Y, sv_b=b)
    for prec in ("double", "single"):
        for sch in ("alternating", "symmetric"):
            s = ref.sinkhorn_solve(X, a, Y, b, eps=0.2, max_iters=40, schedule=sch, precision=prec)
            key = f"sv_{prec[0]}{sch[0]}"
            G[key + "_f"], G[key + "_g"] = s["f_hat"], s["g_hat"]
            G[key + "_s"] = np.array([s["iterations"], s["marginal_violation"], s["dual_cost"],
                                      s["eps"]])
    s = ref.sinkhorn_solve(X, a, Y, b, eps=0.2, max_iters=2000, marginal_tol=1e-9)
    G.update(sv_tol_f=s["f_hat"], sv_tol_g=s["g_hat"],
             sv_tol_s=np.array([s["iterations"], s["marginal_violation"], s["dual_cost"], s["eps"]]))
    s = ref.sinkhorn_solve(X, a, Y, b, eps=0.2, max_iters=300, eps_scaling_factor=0.8,
                           extra_iters_at_final_eps=20)
    G.update(sv_sc_f=s["f_hat"], sv_sc_g=s["g_hat"], sv_sc_hist=s["eps_history"],
             sv_sc_s=np.array([s["iterations"], s["marginal_violation"], s["dual_cost"], s["eps"]]))
    G["sv_div"] = np.array(ref.sinkhorn_divergence(X, a, Y, b, eps=0.2, max_iters=60))

    # fp32 half-step at d = 64 (the tensor-core path's shape class)
    rng = Rng(2024)
    X, a = random_measure(rng, 384, 64)
    Y, b = random_measure(rng, 320, 64)
    g = -0.5 * (Y ** 2).sum(1)
    G.update(f32_X=X, f32_a=a, f32_Y=Y, f32_b=b, f32_g=g,
             f32_out=ref.update_f_hat_f32(X, a, Y, b, g, 0.05),
             f32_out64=ref.update_f_hat(X, a, Y, b, g, 0.05))

    # BASELINE cfg1: n = m = 4096, d = 3, eps = 0.1, 100 alternating iterations,
    # uniform weights, X then Y from fsk::Rng(1000)
    rng = Rng(1000)
    X = np.array([rng.normal() for _ in range(4096 * 3)]).reshape(4096, 3)
    Y = np.array([rng.normal() for _ in range(4096 * 3)]).reshape(4096, 3)
    u = np.full(4096, 1.0 / 4096)
    s = ref.sinkhorn_solve(X, u, Y, u, eps=0.1, max_iters=100)
    G.update(cfg1_X=X, cfg1_Y=Y, cfg1_f=s["f_hat"], cfg1_g=s["g_hat"],
             cfg1_s=np.array([s["iterations"], s["marginal_violation"], s["dual_cost"], s["eps"]]))

    np.savez_compressed(OUT, **G)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(G)} arrays)")


if __name__ == "__main__":
    main()
