"""Top CUDA source lines of an ncu report by stall samples, with the stall-reason split."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
src = open(sys.argv[3]).read().splitlines() if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; res = []
for r in rows:
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0] and r[2] == "-":
        d = dict(zip(hdr, r))
        st = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and v.isdigit() and int(v) > 0}
        res.append((int(d["Warp Stall Sampling (All Samples)"]), int(r[0]), st))
tot = sum(x[0] for x in res) or 1
for n, ln, st in sorted(res, reverse=True)[:top]:
    s = " ".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:4])
    line = src[ln - 1].strip()[:70] if src and ln <= len(src) else ""
    print(f"{n/tot*100:5.1f}% L{ln:<5d} {s:60s} {line}")
