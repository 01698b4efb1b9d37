"""Aggregate a compute-sanitizer racecheck log by (hazard kind, read site, write site)."""
import re
import sys
from collections import Counter

c = Counter()
lines = open(sys.argv[1]).read().splitlines()
for i, l in enumerate(lines):
    m = re.search(r"Potential (\w+) hazard detected at __shared__ (0x[0-9a-f]+)", l)
    if not m:
        continue
    sites = []
    for l2 in lines[i + 1:i + 3]:
        s = re.search(r"(Read|Write) Thread \S+ at (.*?)\+0x[0-9a-f]+ in (\S+)", l2)
        if s:
            sites.append(f"{s.group(1)} {s.group(2)} {s.group(3)}")
    c[(m.group(1),) + tuple(sites)] += 1
for k, v in c.most_common():
    print(v, " | ".join(k))
m = [l for l in lines if "RACECHECK SUMMARY" in l]
print(m[-1] if m else "no summary")
