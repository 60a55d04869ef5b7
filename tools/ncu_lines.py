"""Per-source-line stall attribution from an ncu report (cuda,sass page)."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
res = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        ix = {c: i for i, c in enumerate(hdr)}
        stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or not r or r[0] == "" or len(r) < len(hdr) - 1:
        continue
    v = r[ix["Warp Stall Sampling (All Samples)"]]
    tot = int(v) if v.isdigit() else 0
    if tot:
        br = collections.Counter({c[6:]: int(r[ix[c]]) if r[ix[c]].isdigit() else 0 for c in stalls})
        res.append((tot, r[0], r[1].strip()[:70], br.most_common(3)))
allt = sum(t for t, *_ in res)
for t, ln, src, br in sorted(res, reverse=True)[:top]:
    print(f"{100*t/allt:5.1f}% L{ln:>4} {src:70s} {br}")
