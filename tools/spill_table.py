"""Per-kernel register / spill table from the ptxas logs of a build dir.
  python tools/spill_table.py build/cbessfm [build/cbessfm_base]"""
import re, sys, glob, subprocess
def table(d):
    out = {}
    for f in glob.glob(f"{d}/*.log"):
        cur = None
        for line in open(f):
            m = re.search(r"Function properties for (\S+)", line)
            if m: cur = m.group(1); continue
            m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m and cur: out[cur] = [int(m.group(2)), int(m.group(3))]
            m = re.search(r"Used (\d+) registers", line)
            if m and cur in out: out[cur].append(int(m.group(1))); cur = None
    return out
a = table(sys.argv[1]); b = table(sys.argv[2]) if len(sys.argv) > 2 else {}
names = sorted(a)
dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dm):
    if "block_kernel" not in d and "fat_kernel" not in d and "ip_kernel" not in d: continue
    d = d.replace("cbessfm::", "").replace("(cbessfm::Params<double>)", "").replace("(cbessfm::Params<float>)", "")
    x = a[n]; y = b.get(n)
    if x[0] or (y and y[0]) or len(sys.argv) < 3 or y != x:
        print(f"{d:55s} now st{x[0]:4d} ld{x[1]:4d} r{x[2] if len(x)>2 else '?'}" + (f"   base st{y[0]:4d} ld{y[1]:4d}" if y else ""))
