"""Executed FP32 FLOP/s, L2 and DRAM rates of the dock launches from an ncu metrics CSV
(tools: see DESIGN.md 6).  Usage: fp32_summary.py fp32_ops.csv [submits=4]"""
import collections, csv, sys
path = sys.argv[1]
submits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]; ix = {k: i for i, k in enumerate(h)}
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    per.setdefault((r[ix["ID"]], r[ix["Kernel Name"]]), {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
items = list(per.items()); nl = len(items) // submits; items = items[-nl:]
print("Executed FP32 work of the dock launches (last of %d submits of a 200k C4-shaped library, 6 x 23 bucketing)," % submits)
print("ncu metrics pass (--clock-control none, serialised launches).  flops = FADD + FMUL + 2 FFMA + 2 FADD2 + 2 FMUL2 + 4 FFMA2")
print("(packed FFMA2 = two FMAs).  Peak 74.4 TFLOP/s = 148 SMs x 128 lanes x 2 x 1.965 GHz.\n")
T = F = L = D = 0.0
for (i, name), m in items:
    p = lambda k: m.get(f"sm__sass_thread_inst_executed_op_{k}_pred_on.sum", 0.0)
    fl = p("fadd") + p("fmul") + 2 * p("ffma") + 2 * p("fadd2") + 2 * p("fmul2") + 4 * p("ffma2")
    t = m["gpu__time_duration.sum"] * 1e-9
    dr = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    T += t; F += fl; L += m["lts__t_bytes.sum"]; D += dr
    print(f"{name.split('(')[0].replace('void ', ''):32s} {t * 1e3:7.3f} ms  executed FP32 {fl / t / 1e12:5.2f} TFLOP/s "
          f"({100 * fl / t / 1e12 / 74.45:4.1f}% of peak)  L2 {m['lts__t_bytes.sum'] / t / 1e9:6.1f} GB/s  DRAM {dr / t / 1e9:5.1f} GB/s")
print(f"\nall dock launches: {T * 1e3:.3f} ms, executed FP32 {F / T / 1e12:.2f} TFLOP/s = {100 * F / T / 1e12 / 74.45:.1f}% of the "
      f"FP32 peak; L2 {L / T / 1e9:.1f} GB/s, DRAM {D / T / 1e9:.1f} GB/s (the grid is served from shared memory).")
