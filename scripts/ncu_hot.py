"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
iS, iA, iN = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [(int(r[iA] or 0), r[0], r[iS].strip(), r[iN]) for r in rows[1:] if len(r) > iA]
tot = sum(d[0] for d in data) or 1
for i, (s, a, src, ex) in enumerate(data):
    pass
top = sorted(range(len(data)), key=lambda i: -data[i][0])[:n]
for i in sorted(top):
    s, a, src, ex = data[i]
    print(f"{i:5d} {s/tot:6.1%} exec={ex:>8s}  {src[:90]}")
