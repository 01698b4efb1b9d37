"""Per-source-line cost table from an ncu report (source page, cuda+sass): share of
instructions, shared-memory wavefronts (and their conflict-free ideal) and stall samples."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
src = [r for r in rows[hi + 1:] if len(r) > 5 and r[2] == "-"]
def g(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
T = {k: sum(g(r, k) for r in src) or 1.0 for k in ("Instructions Executed", "L1 Wavefronts Shared", "Warp Stall Sampling (All Samples)")}
print(f"total instructions {T['Instructions Executed']:.4g}  shared wavefronts {T['L1 Wavefronts Shared']:.4g}")
src.sort(key=lambda r: -g(r, "Warp Stall Sampling (All Samples)"))
for r in src[:top]:
    print(f'{r[0]:>4} inst {g(r,"Instructions Executed")/T["Instructions Executed"]*100:5.1f}% '
          f'wf {g(r,"L1 Wavefronts Shared")/T["L1 Wavefronts Shared"]*100:5.1f}% (ideal {g(r,"L1 Wavefronts Shared Ideal")/T["L1 Wavefronts Shared"]*100:5.1f}) '
          f'stall {g(r,"Warp Stall Sampling (All Samples)")/T["Warp Stall Sampling (All Samples)"]*100:5.1f}%  {r[1].strip()[:80]}')
