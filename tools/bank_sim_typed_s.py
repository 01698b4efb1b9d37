"""Bank model (tools/bank_sim3.py) of the TYPED_S corner gathers: window-relative cells of an 18-cell
channel window (fast-path passes only) and a search over row / plane strides (floats)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo/tools'); sys.path.insert(0, '/root/repo')
import bank_sim3 as b
P = b.passes(n=30)
P = P - 7
ok = ((P >= 0) & (P < 18)).all(axis=(1, 2))
P = P[ok][::2]
print("passes", len(P))
print("current (20, 387):", round(b.cost(P, 20, 387), 3))
res = sorted((round(b.cost(P, rs, ps), 3), rs, ps) for rs in range(19, 28) for ps in range(rs * 19, rs * 19 + 33))
print(res[:15])
