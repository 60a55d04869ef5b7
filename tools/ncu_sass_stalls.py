"""Top SASS instructions by one stall reason, with the most recent earlier
load (LDG/LDS/LDTM/LDSM/SHFL) writing one of their source registers.
  python tools/ncu_sass_stalls.py <sass.csv from ncu --page source --print-source=sass> long_sb [top]"""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; ix = {c: i for i, c in enumerate(h)}
reason = "stall_" + sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
ins = [(r[ix["Address"]], r[ix["Source"]].strip(), int(r[ix[reason]] or 0)) for r in rows[2:] if len(r) > 5]
tot = sum(x[2] for x in ins)
print(f"{reason}: {tot} samples")
order = sorted(range(len(ins)), key=lambda i: -ins[i][2])[:top]
regre = re.compile(r"\bR(\d+)\b")
for i in order:
    a, s, n = ins[i]
    srcs = set(regre.findall(s.split(",", 1)[1] if "," in s else ""))
    prod = ""
    for j in range(i - 1, max(0, i - 400), -1):
        t = ins[j][1]
        m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9.]+)\s+R(\d+)", t)
        if m and m.group(3) in srcs and re.match(r"(LDG|LDS|LDTM|LD\.|LDSM|SHFL|LDC|S2R|ATOM|SYNCS)", m.group(2)):
            prod = f"  <- [{i-j:4d} back] {t[:60]}"
            break
    print(f"{n:6d} {100*n/tot:5.1f}% {a[-5:]} {s[:70]:70s}{prod}")
