#!/usr/bin/env python3
"""Probe: can the first g-update (pass 2) skip its 5-MMA screen by bounding its blocks
from the first f-update's gap bounds, transposed? Dense torch reference at n = m = 2^k.

For pass-2 block (Y tile J, X half H) and any j in J, i in H (log2 units):
  t'_ji - M'_j = (t_ij - M_i) + (M_i - L_i + log2 a_i) - (b_j + M'_j)
so  gap'(J, H) <= max_{Jh in J} E1[tile(H), Jh] + max_{i in H}(M_i - L_i + log2 a_i)
                  - min_{j in J} (b_j + M'_j)
with E1 the pass-1 (X tile, Y half) gap bounds and b_j + M'_j = log2 of column j's
largest plan entry after pass 1. Reports the true pass-2 live fraction of (Y tile,
X half) blocks and the bound's, with exact column maxima (the best case), and the
fraction of 'orphan' columns (no live pass-1 block)."""
import math
import sys

import torch


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    n = m = 1 << k
    d, eps, T = 64, 0.05, 26 + k
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(1000)
    X = torch.randn(n, d, device=dev, dtype=torch.float64, generator=g)
    Y = torch.randn(m, d, device=dev, dtype=torch.float64, generator=g)
    L2E = 1.0 / math.log(2.0)
    c = 2.0 / eps * L2E
    loga = math.log2(1.0 / n)
    b = -(Y * Y).sum(1) / eps * L2E + math.log2(1.0 / m)     # pass-1 key bias
    TL = 128
    HL = 64
    nt, nh = n // TL, m // HL
    M = torch.empty(n, device=dev, dtype=torch.float64)
    L = torch.empty(n, device=dev, dtype=torch.float64)
    E1 = torch.empty(nt, nh, device=dev, dtype=torch.float64)
    for r0 in range(0, n, 4096):
        t = c * (X[r0:r0 + 4096] @ Y.T) + b[None, :]
        mx = t.max(1).values
        M[r0:r0 + 4096] = mx
        L[r0:r0 + 4096] = mx + torch.log2(torch.exp2(t - mx[:, None]).sum(1))
        gap = (t - mx[:, None]).view(4096 // TL, TL, nh, HL).amax(dim=(1, 3))
        E1[r0 // TL:(r0 + 4096) // TL] = gap
    live1 = (E1 >= -T).double().mean().item()
    bp = -L + loga                                             # pass-2 key bias (from f)
    # pass 2: rows Y, keys X
    Mp = torch.empty(m, device=dev, dtype=torch.float64)
    nty, nhx = m // TL, n // HL
    E2 = torch.empty(nty, nhx, device=dev, dtype=torch.float64)
    for r0 in range(0, m, 4096):
        t = c * (Y[r0:r0 + 4096] @ X.T) + bp[None, :]
        mx = t.max(1).values
        Mp[r0:r0 + 4096] = mx
        E2[r0 // TL:(r0 + 4096) // TL] = (t - mx[:, None]).view(4096 // TL, TL, nhx, HL).amax(dim=(1, 3))
    live2 = (E2 >= -T).double().mean().item()
    # transposed bound with exact column maxima
    rowterm = (M - L + loga).view(nhx, HL).amax(1)            # per X half
    colterm = (b + Mp).view(nty, TL).amin(1)                  # per Y tile: min_j (b_j + M'_j)
    E1y = E1.view(nt, nty, 2).amax(2)                          # per (X tile, Y tile)
    E1h = E1y.repeat_interleave(2, dim=0)                      # per (X half, Y tile)
    bound = E1h.T + rowterm[None, :] - colterm[:, None]        # (Y tile, X half)
    liveb = (bound >= -T).double().mean().item()
    assert bool((bound >= E2 - 1e-6).all()), "bound violated"
    # orphans: columns with no live pass-1 block (E1 >= -T) in any X tile
    col_live = (E1 >= -T).any(0)                                # per Y half
    orphan_halves = 1.0 - col_live.double().mean().item()
    print(f"n=m=2^{k}: pass-1 live (X tile, Y half) {live1:.4f}; pass-2 true live (Y tile, X half) "
          f"{live2:.4f}; transposed bound live {liveb:.4f}; Y halves with no live pass-1 block "
          f"{orphan_halves:.4f}; colterm spread {float(colterm.max() - colterm.min()):.1f} "
          f"(min {float(colterm.min()):.1f}); rowterm max {float(rowterm.max()):.1f}")


if __name__ == "__main__":
    main()
