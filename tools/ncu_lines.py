"""Per-CUDA-source-line instruction counts and stall samples from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path = None
hdr = None
agg = []
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr and row[0] not in ("", "Function Name") and len(row) == len(hdr):
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            agg.append((path, row[0], row[1], float(row[ie] or 0), float(row[ss] or 0)))
        except ValueError:
            pass
ti = sum(a[3] for a in agg) or 1
ts = sum(a[4] for a in agg) or 1
print(f"total warp instr {ti:.0f}, stall samples {ts:.0f}")
for p, ln, src, ie, ss in sorted(agg, key=lambda a: -a[4])[:top]:
    print(f"{p:16s}:{ln:>4s} instr {ie / ti * 100:5.1f}%  stall {ss / ts * 100:5.1f}%  {src.strip()[:80]}")
