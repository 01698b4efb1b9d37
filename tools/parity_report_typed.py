"""Parity at scale of the TYPED_S layout (Q24): C2 with 4 and with 2 atom types, every ligand and pose
replayed against the fp64 oracle (tools/parity_report.py rows) -> gpurun_out/parity_report_typed_s.json."""
import sys, json, os
sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
import parity_report as p
rows = p.run("C2", 1, True, typed=4) + p.run("C2", 1, True, typed=2)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"band": p.BAND, "tol_score": p.TOL_S, "tol_xyz": p.TOL_X, "layout": "TYPED_S (scalar channel windows)", "rows": rows},
          open("gpurun_out/parity_report_typed_s.json", "w"), indent=1)
print(json.dumps(rows)[:2000])
