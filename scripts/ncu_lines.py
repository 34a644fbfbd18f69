"""Per-CUDA-line instruction counts / stall samples from an ncu report (cuda,sass view)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 8 and r[0] and r[0] != "Line No" and r[2] == "-":
        try:
            res.append((int(r[7]), int(r[4]), fname, r[0], r[1][:110]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
for n, st, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{n/tot*100:5.1f}% stall {st:8d} {f}:{ln:5s} {src}")
