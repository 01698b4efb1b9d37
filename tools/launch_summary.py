"""Summarise an ncu launch list (gpu__time_duration + dram bytes per kernel) of bench.py --steps 1 --warmup 1.
Writes the per-step dock-phase DRAM traffic to profiles/dock_traffic.json (read by bench.py's roofline)."""
import collections, csv, json, sys
path, out_json = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
rows = list(csv.reader(open(path)))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"])
    per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, name), m in per.items():
    short = name.split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("dk::", "").replace("vsd::", "")
    a = agg[short]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
# bench.py's live roofline denominators (tools/ceilings.cu: k_l2, k_gather) and torch's own
# kernels run outside the timed step: listed, not counted in the step's shares
EXTERNAL = ("k_l2", "k_gather", "at::")
tot = sum(a[1] for k, a in agg.items() if not k.lstrip("<").startswith(EXTERNAL))
print(f"{'launches':>8} {'time_ms':>10} {'share':>7} {'dram_MB':>10}  kernel   (2 steps: warmup + timed; ncu serialised, cold cache)")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    ext = k.lstrip("<").startswith(EXTERNAL)
    share = "   ext" if ext else f"{100*a[1]/tot:5.1f}%"
    print(f"{a[0]:8d} {a[1]/1e6:10.3f} {share:>7} {a[2]/1e6:10.1f}  {k}")
dock = [v for k, v in agg.items() if k.startswith("dock_kernel")]
steps = 2
if out_json:
    n_l = sum(v[0] for v in dock) / steps
    json.dump({"config": "C4", "n": 1000000, "source": path, "steps_in_capture": steps,
               "dock_launches_per_step": n_l,
               "dram_bytes_per_dock_phase": sum(v[2] for v in dock) / steps,
               "dram_bytes_per_dock_launch": sum(v[2] for v in dock) / max(1, sum(v[0] for v in dock)),
               "dock_share_of_step": sum(v[1] for v in dock) / tot}, open(out_json, "w"), indent=1)
