"""Per-source-line memory traffic from an ncu report: L1 shared wavefronts
and global-load sectors/requests (cuda,sass source page)."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
res = []
def iv(x):
    x = x.replace(",", "")
    return int(float(x)) if x.replace(".", "").isdigit() else 0
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        ix = {c: i for i, c in enumerate(hdr)}
        continue
    if hdr is None or not r or r[0] == "" or len(r) < len(hdr) - 1:
        continue
    sh = iv(r[ix["L1 Wavefronts Shared"]])
    gs = iv(r[ix["L2 Theoretical Sectors Global"]])
    greq = iv(r[ix["L1 Tag Requests Global"]])
    if sh or gs or greq:
        res.append((sh + gs, sh, gs, greq, r[0], r[1].strip()[:80]))
tsh = sum(x[1] for x in res); tgs = sum(x[2] for x in res); treq = sum(x[3] for x in res)
print(f"total shared wavefronts {tsh:.3e}, global sectors {tgs:.3e}, global requests {treq:.3e}")
for tot, sh, gs, greq, ln, src in sorted(res, reverse=True)[:top]:
    print(f"L{ln:>4} sh {sh:>10d} gsec {gs:>10d} greq {greq:>9d}  {src}")
