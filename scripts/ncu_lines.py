"""Per-source-line warp-stall summary of an ncu report (source page, cuda+sass):
python scripts/ncu_lines.py REPORT.ncu-rep [first_line last_line] [--file ace_hash_tc.cu]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10**9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
S = hdr.index("Warp Stall Sampling (All Samples)")
I = hdr.index("Instructions Executed")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg, src, fname = {}, {}, ""
for r in rows:
    if not r or r[0] in ("Function Name", "Line No"):
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "":
        continue
    key = (fname, int(r[0]))
    src[key] = r[1].strip()[:80]
    try:
        agg[key] = [int(r[S]), int(r[I])] + [int(r[i] or 0) for i, _ in reasons]
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values())
print(f"samples {tot} instructions {sum(v[1] for v in agg.values())}")
sel = [(k, v) for k, v in agg.items() if lo <= k[1] <= hi]
for k, v in sorted(sel, key=lambda kv: -kv[1][0])[:40]:
    top = sorted(((v[2 + j], h[6:]) for j, (_, h) in enumerate(reasons)), reverse=True)[:3]
    print(f"{k[0][:14]:14s}:{k[1]:4d} {v[0]:6d} {100 * v[0] / max(tot, 1):5.1f}% ins {v[1]:9d} "
          + " ".join(f"{n}={c}" for c, n in top if c) + f" | {src[k]}")
