import re, sys
cur = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "paper_2303_06150_b200/build.log"):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1); continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        k = re.search(r"dock_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELb(\d)", cur)
        name = (f"dock AC={k.group(1)} NW={k.group(2)} PPW={k.group(3)} GM={k.group(4)} K={k.group(5)} MS={k.group(6)}"
                if k else re.sub(r"_ZN3vsd\w+?_\d+", "", cur)[:60])
        print(name, "regs", m.group(1), line.strip().split("registers,")[-1])
        cur = None
    if "spill" in line and not line.strip().startswith("0 bytes stack frame, 0 bytes spill stores, 0 bytes spill loads"):
        print("   ", line.strip())
